// mma_rate_probe.cu -- dev probe: cycles per tcgen05.mma.cta_group::1.kind::i8 (M = 128, K = 32)
// issued back to back into one accumulator, A from TMEM ("TS") or from shared memory ("SS"),
// for several N. Answers whether small-N MMAs are bound by the A-operand read rather than by
// the N-proportional floor (K6 issues M=128, N=16..80 MMAs).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/mma_rate_probe scripts/mma_rate_probe.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t desc_sw128(uint32_t a) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((a >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>(1) << 16;
  d |= static_cast<uint64_t>(1024 >> 4) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(2) << 61;
  return d;
}
__host__ __device__ constexpr uint32_t idesc(uint32_t M, uint32_t N) {
  return (2u << 4) | ((N >> 3) << 17) | ((M >> 4) << 24);
}

template <int N, bool TS, bool STORE = false, int ND = 1>
__global__ void probe(unsigned long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x01010101u;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t t = tbase;
  if (threadIdx.x == 0) {
    const uint32_t a_smem = su32(smem), b_smem = su32(smem + 32 * 1024);
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const uint32_t k = i & 3;
      const uint64_t bd = desc_sw128(b_smem + k * 32);
      if (TS) {
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(t + 256 + (i % ND) * 64),
                     "r"(t + (i & 15) * 8), "l"(bd), "r"(idesc(128, N)), "r"(i >= ND ? 1 : 0));
      } else {
        const uint64_t ad = desc_sw128(a_smem + k * 32);
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(t + 256 + (i % ND) * 64),
                     "l"(ad), "l"(bd), "r"(idesc(128, N)), "r"(i >= ND ? 1 : 0));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
    asm volatile("{\n\t.reg .pred P1;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W;\n\t}" ::"r"(su32(&bar)) : "memory");
    out[blockIdx.x] = clock64() - t0;
  } else if (STORE && threadIdx.x >= 32) {
    // warps 1..3: tcgen05.st 32x32b.x32 into their lane quarter, columns 384.., for as long as
    // the MMAs run (the K6 transform warps' traffic next to the MMA's A-operand reads)
    const uint32_t w = threadIdx.x >> 5;
    uint32_t r[32];
    for (int i = 0; i < 32; ++i) r[i] = threadIdx.x * 33u + i;
    const uint32_t addr = t + ((32u * w) << 16) + 384u;
    for (int it = 0; it < iters / 4; ++it) {
      asm volatile(
          "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, "
          "%13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(addr),
          "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
          "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
          "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
          "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
          : "memory");
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(t));
}

template <int N, bool TS, bool STORE = false, int ND = 1>
void run(unsigned long long* d, int sms) {
  auto k = probe<N, TS, STORE, ND>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  const int iters = 4096;
  k<<<sms, 128, 100 * 1024>>>(d, iters);
  k<<<sms, 128, 100 * 1024>>>(d, iters);
  unsigned long long h[256];
  cudaMemcpy(h, d, sms * 8, cudaMemcpyDeviceToHost);
  double s = 0;
  for (int i = 0; i < sms; ++i) s += h[i];
  std::printf("%s%s N=%3d, %d accumulators: %6.1f cycles per MMA (M=128 K=32; all %d SMs busy) err=%s\n",
              TS ? "TS" : "SS", STORE ? " + concurrent tcgen05.st (3 warps)" : "", N, ND,
              s / sms / iters, sms, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* d;
  cudaMalloc(&d, 256 * 8);
  run<16, true>(d, sms);
  run<32, true>(d, sms);
  run<64, true>(d, sms);
  run<128, true>(d, sms);
  run<256, true>(d, sms);
  run<16, false>(d, sms);
  run<32, false>(d, sms);
  run<64, false>(d, sms);
  run<128, false>(d, sms);
  run<256, false>(d, sms);
  run<32, true, true>(d, sms);
  run<64, true, true>(d, sms);
  run<32, false, true>(d, sms);
  run<32, true, false, 2>(d, sms);
  run<32, true, false, 4>(d, sms);
  run<32, false, false, 2>(d, sms);
  run<64, true, false, 2>(d, sms);
  return 0;
}
