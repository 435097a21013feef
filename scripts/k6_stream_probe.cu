// k6_stream_probe.cu -- dev probe: K6's weight-stream access pattern alone (no math), graph
// chain over rotating weight copies. 148 CTAs x 16 warps; the tile-steps (128 rows x 512
// columns of a W3 8192 x 8192 plane tensor) are dealt as contiguous ranges; warp (rg, set)
// loads the 16-row slice of its set's steps through a one-slot ring and touches it.
//   pair = 0: box {16 words, 16 rows, 3 planes} per step (K6 as shipped, 64-byte row segments)
//   pair = 1: box {32 words, 16 rows, 3 planes} per step pair (128-byte row segments, sets own
//             pairs of consecutive steps)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/k6_stream_probe scripts/k6_stream_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                 \
  do {                                                                        \
    cudaError_t e_ = (x);                                                     \
    if (e_ != cudaSuccess) {                                                  \
      std::printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      std::exit(1);                                                           \
    }                                                                         \
  } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

struct P {
  uint32_t total, spt, pair, work;
  int* out;
};

__global__ void __launch_bounds__(512, 1) k6s(const __grid_constant__ CUtensorMap tm, const P p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar[16];
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t q = warp & 3, h = warp >> 2, rg = 2 * q + (h & 1), set = h >> 1;
  const uint32_t box = p.pair ? 6144u : 3072u;
  if (lane == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[warp])));
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncwarp();
  const uint32_t a = uint64_t(blockIdx.x) * p.total / gridDim.x;
  const uint32_t b = uint64_t(blockIdx.x + 1) * p.total / gridDim.x;
  const uint32_t stride = p.pair ? 4u : 2u, own = p.pair ? 2u * set : set;
  auto issue = [&](uint32_t j) {
    if (j < b && lane == 0) {
      const uint32_t tile = j / p.spt, s = j % p.spt;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[warp])), "r"(box) : "memory");
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(su32(smem + warp * 6144)),
          "l"(reinterpret_cast<uint64_t>(&tm)), "r"(su32(&bar[warp])), "r"(int(s * 16)),
          "r"(int(tile * 128 + rg * 16)), "r"(0)
          : "memory");
    }
  };
  asm volatile("griddepcontrol.wait;" ::: "memory");
  uint32_t acc = 0, ph = 0;
  uint32_t j = a + own;
  issue(j);
  for (; j < b; j += stride) {
    asm volatile(
        "{\n\t.reg .pred P1;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra W_%=;\n\t}" ::"r"(su32(&bar[warp])), "r"(ph) : "memory");
    ph ^= 1u;
    acc += reinterpret_cast<const uint32_t*>(smem + warp * 6144)[lane];
    __syncwarp();
    issue(j + stride);
    if (p.work) {
      const long long t0 = clock64();
      while (clock64() - t0 < p.work) acc = acc * 3u + 1u;
    }
  }
  asm volatile("griddepcontrol.launch_dependents;");
  if (acc == 0x12345678u) p.out[0] = acc;
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
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, s);
  for (int r = 0; r < 5; ++r) CK(cudaGraphLaunch(ge, s));
  cudaEventRecord(e1, s);
  CK(cudaStreamSynchronize(s));
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms * 1e3f / (5 * reps);
}

int main() {
  cudaStream_t s;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  int* out;
  CK(cudaMalloc(&out, 64));
  const uint32_t rows = 8192, wpr = 256, np = 3;
  const uint64_t bytes = uint64_t(np) * rows * wpr * 4;
  const int nbuf = static_cast<int>(300e6 / bytes) + 2;
  std::vector<uint8_t*> bufs(nbuf);
  for (auto& b : bufs) {
    CK(cudaMalloc(&b, bytes));
    CK(cudaMemset(b, 1, bytes));
  }
  for (uint32_t pair = 0; pair < 2; ++pair) {
    for (uint32_t work : {0u, 1500u}) {
      std::vector<CUtensorMap> tms(nbuf);
      for (int i = 0; i < nbuf; ++i) {
        const cuuint64_t d[3] = {wpr, rows, np};
        const cuuint64_t st[2] = {uint64_t(wpr) * 4, uint64_t(wpr) * 4 * rows};
        const cuuint32_t bx[3] = {pair ? 32u : 16u, 16, np};
        const cuuint32_t es[3] = {1, 1, 1};
        if (cuTensorMapEncodeTiled(&tms[i], CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, bufs[i], d, st, bx, es,
                                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
          std::printf("encode failed\n");
          return 1;
        }
      }
      const uint32_t spt = pair ? 8 : 16;  // steps per tile in units of the box
      const uint32_t total = (rows / 128) * spt;
      CK(cudaFuncSetAttribute(k6s, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
      const float us = graph_us(s, 40, [&](int i) {
        P pp{total, spt, pair, work, out};
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(148);
        cfg.blockDim = dim3(512);
        cfg.dynamicSmemBytes = 200 * 1024;
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        CK(cudaLaunchKernelEx(&cfg, k6s, tms[i % nbuf], pp));
      });
      std::printf("K6 stream pattern, W3 8192^2 (25.2 MB), %s, %u cycles/item: %6.2f us/call %5.0f GB/s\n",
                  pair ? "32-word boxes per step pair" : "16-word boxes per step", work, us, bytes / us / 1e3);
    }
  }
  return 0;
}
