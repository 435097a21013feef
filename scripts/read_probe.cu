// Microbenchmark: how fast can one kernel stream N bytes from HBM on this GPU (the
// practical HBM roofline for the skinny path's sizes, incl. launch + ramp).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o read_probe read_probe.cu
#include <cstdio>
#include <cstdint>
__global__ void rd(const uint4* __restrict__ p, size_t n16, uint32_t* out) {
  uint32_t acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p + i));
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x12345678u) out[0] = acc;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  size_t maxb = size_t(1) << 30;
  uint4* buf; cudaMalloc(&buf, maxb * 2);  // two regions: alternate to defeat L2 reuse
  uint32_t* out; cudaMalloc(&out, 4);
  cudaMemset(buf, 1, maxb * 2);
  for (size_t mb : {4, 11, 25, 50, 100, 201, 1024}) {
    size_t bytes = mb << 20, n16 = bytes / 16;
    for (int bpsm : {4, 8, 16}) {
      int grid = sms * bpsm;
      for (int i = 0; i < 3; ++i) rd<<<grid, 256>>>(buf, n16, out);
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      const int reps = 40;
      cudaEventRecord(e0);
      for (int i = 0; i < reps; ++i) rd<<<grid, 256>>>(buf + (i & 1) * (maxb / 16), n16, out);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double us = 1e3 * ms / reps;
      printf("%5zu MB  blocks/SM=%2d  %8.2f us  %7.0f GB/s\n", mb, bpsm, us, bytes / us / 1e3);
    }
  }
  return 0;
}
