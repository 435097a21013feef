// stream_floor.cu -- dev probe: what a back-to-back chain of HBM-streaming kernels costs per
// call on this part (CUDA graph replay, the serving pattern), independent of any GEMM math.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/stream_floor scripts/stream_floor.cu -lcuda
//   scripts/stream_floor
// Variants: empty kernels (launch floor), and a stream kernel in which every CTA bulk-copies
// its contiguous share of a buffer through a shared-memory ring (one producer thread, the
// consumer warps touch each chunk), with the PDL trigger / early loads on or off and the
// ring size (co-residency of the next call's CTAs) varied.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>

#define CK(x)                                                                       \
  do {                                                                              \
    cudaError_t e_ = (x);                                                           \
    if (e_ != cudaSuccess) {                                                        \
      std::printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));       \
      std::exit(1);                                                                 \
    }                                                                               \
  } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" :::); }

__global__ void empty_kernel(int* out, int pdl) {
  if (pdl) {
    pdl_trigger();
    pdl_wait();
  }
  if (threadIdx.x == 0 && blockIdx.x == 100000) out[0] = 1;
}

struct SP {
  const uint8_t* src;
  uint64_t bytes_per_cta;
  uint32_t chunk, slots;
  uint32_t early;    // issue the first loads before griddepcontrol.wait
  uint32_t trigger;  // 0: at end, 1: at start
  int* out;
};

// block: 1 producer warp + C consumer warps
__global__ void stream_kernel(const SP p) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[32], empty[32];
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t cons = blockDim.x / 32 - 1;
  if (p.trigger) pdl_trigger();
  if (threadIdx.x == 0) {
    for (uint32_t s = 0; s < p.slots; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&empty[s])), "r"(cons));
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  const uint8_t* base = p.src + uint64_t(blockIdx.x) * p.bytes_per_cta;
  const uint32_t n = static_cast<uint32_t>(p.bytes_per_cta / p.chunk);
  if (warp == 0) {
    if (lane == 0) {
      if (!p.early) pdl_wait();
      for (uint32_t i = 0; i < n; ++i) {
        const uint32_t s = i % p.slots;
        if (i >= p.slots) {
          const uint32_t par = ((i / p.slots) - 1) & 1;
          asm volatile(
              "{\n\t.reg .pred P1;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
              "@!P1 bra W_%=;\n\t}" ::"r"(su32(&empty[s])), "r"(par) : "memory");
        }
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])),
                     "r"(p.chunk) : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                su32(smem + s * p.chunk)),
            "l"(base + uint64_t(i) * p.chunk), "r"(p.chunk), "r"(su32(&full[s]))
            : "memory");
      }
    }
  } else {
    pdl_wait();
    uint32_t acc = 0;
    for (uint32_t i = 0; i < n; ++i) {
      const uint32_t s = i % p.slots;
      const uint32_t par = (i / p.slots) & 1;
      asm volatile(
          "{\n\t.reg .pred P1;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
          "@!P1 bra W_%=;\n\t}" ::"r"(su32(&full[s])), "r"(par) : "memory");
      const uint32_t* w = reinterpret_cast<const uint32_t*>(smem + s * p.chunk);
      for (uint32_t q = (warp - 1) * 32 + lane; q < p.chunk / 4; q += cons * 32 * 8) acc += w[q];
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[s])) : "memory");
    }
    if (acc == 0x12345678u) p.out[0] = acc;
  }
  if (!p.trigger) pdl_trigger();
}


struct TP {
  uint32_t bw, br, np, kchunks, total_items;
  uint32_t slots, box_bytes;
  int* out;
};
// tensor-map variant: items (row tile, K chunk) of a [np][rows][wpr] u32 plane tensor, box
// {bw words, br rows, np planes}; CTA c takes items [c*total/grid, (c+1)*total/grid)
__global__ void tstream_kernel(const __grid_constant__ CUtensorMap tm, const TP p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[32], empty[32];
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t cons = blockDim.x / 32 - 1;
  pdl_trigger();
  if (threadIdx.x == 0) {
    for (uint32_t s = 0; s < p.slots; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&empty[s])), "r"(cons));
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  const uint32_t i0 = uint64_t(blockIdx.x) * p.total_items / gridDim.x;
  const uint32_t i1 = uint64_t(blockIdx.x + 1) * p.total_items / gridDim.x;
  const uint32_t n = i1 - i0;
  if (warp == 0) {
    if (lane == 0) {
      for (uint32_t i = 0; i < n; ++i) {
        const uint32_t s = i % p.slots;
        if (i >= p.slots) {
          const uint32_t par = ((i / p.slots) - 1) & 1;
          asm volatile(
              "{\n\t.reg .pred P1;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
              "@!P1 bra W_%=;\n\t}" ::"r"(su32(&empty[s])), "r"(par) : "memory");
        }
        const uint32_t it = i0 + i, tile = it / p.kchunks, kc = it % p.kchunks;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])),
                     "r"(p.box_bytes) : "memory");
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(su32(smem + s * p.box_bytes)),
            "l"(reinterpret_cast<uint64_t>(&tm)), "r"(su32(&full[s])), "r"(int(kc * p.bw)),
            "r"(int(tile * p.br)), "r"(0)
            : "memory");
      }
    }
  } else {
    pdl_wait();
    uint32_t acc = 0;
    for (uint32_t i = 0; i < n; ++i) {
      const uint32_t s = i % p.slots;
      const uint32_t par = (i / p.slots) & 1;
      asm volatile(
          "{\n\t.reg .pred P1;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
          "@!P1 bra W_%=;\n\t}" ::"r"(su32(&full[s])), "r"(par) : "memory");
      const uint32_t* w = reinterpret_cast<const uint32_t*>(smem + s * p.box_bytes);
      for (uint32_t q = (warp - 1) * 32 + lane; q < p.box_bytes / 4; q += cons * 32 * 8) acc += w[q];
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[s])) : "memory");
    }
    if (acc == 0x12345678u) p.out[0] = acc;
  }
}

template <typename F>
float graph_us(cudaStream_t s, int reps, F launch) {
  cudaGraph_t g;
  cudaGraphExec_t ge;
  for (int i = 0; i < 3; ++i) launch(i);
  CK(cudaStreamSynchronize(s));
  CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal));
  for (int i = 0; i < reps; ++i) launch(i);
  CK(cudaStreamEndCapture(s, &g));
  CK(cudaGraphInstantiate(&ge, g, 0));
  CK(cudaGraphLaunch(ge, s));
  CK(cudaStreamSynchronize(s));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a, s);
  for (int r = 0; r < 5; ++r) CK(cudaGraphLaunch(ge, s));
  cudaEventRecord(b, s);
  CK(cudaStreamSynchronize(s));
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  cudaGraphExecDestroy(ge);
  cudaGraphDestroy(g);
  return ms * 1e3f / (5 * reps);
}

int main() {
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaStream_t s;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  int* out;
  CK(cudaMalloc(&out, 64));
  const int reps = 40;
  for (int pdl = 0; pdl < 2; ++pdl) {
    for (int thr : {128, 512}) {
      const float us = graph_us(s, reps, [&](int) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(sms);
        cfg.blockDim = dim3(thr);
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = pdl;
        CK(cudaLaunchKernelEx(&cfg, empty_kernel, out, pdl));
      });
      std::printf("empty kernel grid %d x %d threads, pdl %d: %.2f us/call\n", sms, thr, pdl, us);
    }
  }
  // stream kernels over `nbuf` rotating buffers so nothing stays in L2
  for (double mb : {4.2, 25.2, 50.3}) {
    const uint64_t per_cta = (static_cast<uint64_t>(mb * 1e6 / sms) + 16383) / 16384 * 16384;
    const uint64_t bytes = per_cta * sms;
    const int nbuf = static_cast<int>(400e6 / bytes) + 2;
    std::vector<uint8_t*> bufs(nbuf);
    for (auto& b : bufs) {
      CK(cudaMalloc(&b, bytes));
      CK(cudaMemset(b, 1, bytes));
    }
    struct V { uint32_t chunk, slots, early, trigger, pdl, threads; };
    const V vs[] = {
        {16384, 12, 0, 0, 0, 160}, {16384, 12, 0, 0, 1, 160}, {16384, 12, 1, 0, 1, 160},
        {16384, 12, 1, 1, 1, 160}, {16384, 6, 1, 1, 1, 160},  {8192, 12, 1, 1, 1, 160},
        {16384, 6, 0, 0, 1, 160},  {4096, 24, 1, 1, 1, 160},  {16384, 6, 1, 1, 1, 288},
    };
    for (const V& v : vs) {
      const uint32_t sm = v.chunk * v.slots;
      CK(cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
      const float us = graph_us(s, reps, [&](int i) {
        SP p{bufs[i % nbuf], per_cta, v.chunk, v.slots, v.early, v.trigger, out};
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(sms);
        cfg.blockDim = dim3(v.threads);
        cfg.dynamicSmemBytes = sm;
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = v.pdl;
        CK(cudaLaunchKernelEx(&cfg, stream_kernel, p));
      });
      std::printf("stream %5.1f MB chunk %5u x %2u slots (%3u KB) thr %3u early %u trig_start %u pdl %u: "
                  "%6.2f us/call  %5.0f GB/s\n",
                  bytes / 1e6, v.chunk, v.slots, sm / 1024, v.threads, v.early, v.trigger, v.pdl, us,
                  bytes / us / 1e3);
    }
    for (auto& b : bufs) cudaFree(b);
  }

  // tensor-map item shapes over a W3 8192 x 8192 plane tensor (25.2 MB) and W2 4096^2
  for (int shape = 0; shape < 2; ++shape) {
    const uint32_t rows = shape == 0 ? 8192 : 4096, wpr = rows / 32, np = shape == 0 ? 3 : 2;
    const uint64_t bytes = uint64_t(np) * rows * wpr * 4;
    const int nbuf = static_cast<int>(400e6 / bytes) + 2;
    std::vector<uint8_t*> bufs(nbuf);
    std::vector<CUtensorMap> tms(nbuf);
    struct B { uint32_t bw, br, ring_kb, threads; };
    const B bs[] = {{16, 16, 96, 160}, {64, 16, 96, 160}, {128, 16, 96, 160}, {256, 16, 96, 160},
                    {256, 8, 96, 160},  {32, 32, 96, 160}, {64, 32, 96, 160},  {128, 8, 96, 160},
                    {16, 16, 192, 544}, {128, 16, 192, 160}};
    for (auto& b : bufs) {
      CK(cudaMalloc(&b, bytes));
      CK(cudaMemset(b, 1, bytes));
    }
    for (const B& b : bs) {
      if (b.bw > wpr) continue;
      for (int i = 0; i < nbuf; ++i) {
        const cuuint64_t d[3] = {wpr, rows, np};
        const cuuint64_t st[2] = {uint64_t(wpr) * 4, uint64_t(wpr) * 4 * rows};
        const cuuint32_t bx[3] = {b.bw, b.br, np};
        const cuuint32_t es[3] = {1, 1, 1};
        if (cuTensorMapEncodeTiled(&tms[i], CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, bufs[i], d, st, bx, es,
                                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
          std::printf("encode failed\n");
          return 1;
        }
      }
      const uint32_t box_bytes = b.bw * b.br * np * 4;
      const uint32_t slots = std::min<uint32_t>(32, b.ring_kb * 1024 / box_bytes);
      const uint32_t sm = slots * box_bytes;
      CK(cudaFuncSetAttribute(tstream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, sm + 1024));
      const uint32_t kchunks = wpr / b.bw, total = (rows / b.br) * kchunks;
      const float us = graph_us(s, reps, [&](int i) {
        TP p{b.bw, b.br, np, kchunks, total, slots, box_bytes, out};
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(sms);
        cfg.blockDim = dim3(b.threads);
        cfg.dynamicSmemBytes = sm + 1024;
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        CK(cudaLaunchKernelEx(&cfg, tstream_kernel, tms[i % nbuf], p));
      });
      std::printf("tmap %5.1f MB box {%3u words, %2u rows, %u planes} = %5u B x %2u slots thr %3u: "
                  "%6.2f us/call  %5.0f GB/s\n", bytes / 1e6, b.bw, b.br, np, box_bytes, slots,
                  b.threads, us, bytes / us / 1e3);
    }
    for (auto& b : bufs) cudaFree(b);
  }
  return 0;
}
