// Microbenchmark: legacy-pipe mma.sync m16n8k32 u8 (IMMA.16832) throughput on this GPU.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o imma_probe imma_probe.cu
#include <cstdio>
#include <cstdint>
__global__ void probe(uint32_t* out, int iters) {
  uint32_t d[8][4] = {};
  uint32_t a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 ^ 0x55, b1 = a0 ^ 0x33;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < 8; ++c)
      asm volatile(
          "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
          "{%0,%1,%2,%3};"
          : "+r"(d[c][0]), "+r"(d[c][1]), "+r"(d[c][2]), "+r"(d[c][3])
          : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  uint32_t s = 0;
  for (int c = 0; c < 8; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  uint32_t* out; cudaMalloc(&out, 1 << 24);
  const int iters = 4096;
  for (int warps : {4, 8, 16, 32}) {
    probe<<<sms, warps * 32>>>(out, 16);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    probe<<<sms, warps * 32>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double mmas = double(sms) * warps * iters * 8;
    double macs = mmas * 16 * 8 * 32;
    printf("warps/SM=%2d: %.3f ms, %.1f TOPS (2*MAC), %.2f MMA/clk/SM at %d MHz\n", warps, ms,
           2 * macs / ms / 1e9, mmas / sms / (ms * 1e-3 * clk * 1e3), clk / 1000);
  }
  return 0;
}
