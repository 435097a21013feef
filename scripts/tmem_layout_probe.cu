// tmem_layout_probe.cu -- dev probe: where tcgen05.st.16x256b puts each thread's registers.
// Thread T stores value (T << 8) | i from register i with .16x256b.x2 at lane base 0, column
// 0, then every thread reads its lane back with .32x32b.x16; prints (lane, column) -> (T, i).
//   nvcc -gencode arch=compute_100a,code=sm_100a -o scripts/tmem_layout_probe scripts/tmem_layout_probe.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__global__ void probe(uint32_t* out) {
  __shared__ uint32_t base_s;
  const uint32_t t = threadIdx.x;
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(
      static_cast<uint32_t>(__cvta_generic_to_shared(&base_s))));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t base = base_s;
  uint32_t v[8];
  for (int i = 0; i < 8; ++i) v[i] = (t << 8) | i;
  asm volatile("tcgen05.st.sync.aligned.16x256b.x2.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(base),
               "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
               : "memory");
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
      "%12, %13, %14, %15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(base));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  for (int i = 0; i < 16; ++i) out[t * 16 + i] = r[i];
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(base));
}

int main() {
  uint32_t* d;
  cudaMalloc(&d, 32 * 16 * 4);
  cudaMemset(d, 0xff, 32 * 16 * 4);
  probe<<<1, 32>>>(d);
  uint32_t h[32 * 16];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  std::printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  for (int lane = 0; lane < 16; ++lane) {
    std::printf("lane %2d:", lane);
    for (int c = 0; c < 16; ++c) {
      const uint32_t x = h[lane * 16 + c];
      std::printf(" %2u.%u", x >> 8, x & 0xff);
    }
    std::printf("\n");
  }
  return 0;
}
