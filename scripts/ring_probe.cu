// ring_probe.cu -- dev probe: the decode kernel's (K5) weight-streaming skeleton alone, in a
// CUDA-graph chain of back-to-back calls over rotating weight copies (the serving pattern).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/ring_probe scripts/ring_probe.cu -lcuda
//   scripts/ring_probe
// Each of 16 warps per CTA owns a ring of `stages` TMA slots and walks its items exactly as
// skinny_kernel does (one 64-row tile per CTA, four K groups of warps, items of 16 rows x
// `bw` words x n planes). No GEMM math: a consumer touches one word per item and optionally
// spins `work` cycles per item (the transposes + MMAs) and `delay` cycles after the PDL
// wait (the feature staging). Answers: does a 128-byte row segment (bw = 32) stream better
// than 64 bytes (bw = 16), what does the ring depth do, and what do the staging delay and
// the per-item work cost on top of the stream.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e_ = (x);                                                      \
    if (e_ != cudaSuccess) {                                                   \
      std::printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));  \
      std::exit(1);                                                            \
    }                                                                          \
  } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

struct P {
  uint32_t bw, np, stages, cpw, delay, work, box_bytes;
  int* out;
};

__global__ void __launch_bounds__(512, 1) ring_kernel(const __grid_constant__ CUtensorMap tm, const P p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t bars[16 * 8];
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t wr = warp >> 2, wk = warp & 3u;
  uint64_t* mb = bars + warp * 8;
  const uint32_t ring = su32(smem) + warp * p.stages * p.box_bytes;
  if (lane == 0) {
    for (uint32_t s = 0; s < p.stages; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&mb[s])));
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncwarp();
  const uint32_t row0 = blockIdx.x * 64u + wr * 16u;
  uint32_t is_c = 0;
  auto issue = [&](uint32_t slot) {
    if (is_c < p.cpw && lane == 0) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&mb[slot])),
                   "r"(p.box_bytes) : "memory");
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(ring + slot * p.box_bytes),
          "l"(reinterpret_cast<uint64_t>(&tm)), "r"(su32(&mb[slot])), "r"(int((is_c * 4 + wk) * p.bw)),
          "r"(int(row0)), "r"(0)
          : "memory");
    }
    ++is_c;
  };
  for (uint32_t s = 0; s + 1 < p.stages; ++s) issue(s);
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (p.delay) {
    const long long t0 = clock64();
    while (clock64() - t0 < p.delay) {
    }
  }
  __syncthreads();
  uint32_t acc = 0, phase = 0;
  for (uint32_t c = 0; c < p.cpw; ++c) {
    __syncwarp();
    issue((c + p.stages - 1) % p.stages);
    const uint32_t slot = c % p.stages;
    asm volatile(
        "{\n\t.reg .pred P1;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra W_%=;\n\t}" ::"r"(su32(&mb[slot])), "r"((phase >> slot) & 1u) : "memory");
    phase ^= 1u << slot;
    acc += reinterpret_cast<const uint32_t*>(smem + warp * p.stages * p.box_bytes + slot * p.box_bytes)[lane];
    if (p.work) {
      const long long t0 = clock64();
      while (clock64() - t0 < p.work) acc = acc * 3u + 1u;
    }
    if (c + 1 == p.cpw) asm volatile("griddepcontrol.launch_dependents;");
  }
  __syncthreads();
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
  cudaStream_t s;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  int* out;
  CK(cudaMalloc(&out, 64));
  const uint32_t rows = 8192, wpr = 256, np = 3;
  const uint64_t bytes = uint64_t(np) * rows * wpr * 4;  // 25.2 MB, W3 8192 x 8192
  const int nbuf = static_cast<int>(300e6 / bytes) + 2;
  std::vector<uint8_t*> bufs(nbuf);
  for (auto& b : bufs) {
    CK(cudaMalloc(&b, bytes));
    CK(cudaMemset(b, 1, bytes));
  }
  struct V { uint32_t bw, stages, delay, work, smem_kb; };
  const V vs[] = {
      {16, 2, 0, 0, 224},    {32, 2, 0, 0, 224},    {16, 3, 0, 0, 224},    {16, 4, 0, 0, 224},
      {16, 2, 4000, 0, 224}, {32, 2, 4000, 0, 224}, {16, 4, 4000, 0, 224},
      {16, 2, 0, 800, 224},  {32, 2, 0, 1600, 224}, {16, 4, 0, 800, 224},  {16, 2, 4000, 800, 224},
      {32, 2, 4000, 1600, 224}, {16, 4, 4000, 800, 224}, {16, 2, 0, 0, 100}, {16, 2, 4000, 800, 100},
  };
  for (const V& v : vs) {
    std::vector<CUtensorMap> tms(nbuf);
    for (int i = 0; i < nbuf; ++i) {
      const cuuint64_t d[3] = {wpr, rows, np};
      const cuuint64_t st[2] = {uint64_t(wpr) * 4, uint64_t(wpr) * 4 * rows};
      const cuuint32_t bx[3] = {v.bw, 16, np};
      const cuuint32_t es[3] = {1, 1, 1};
      if (cuTensorMapEncodeTiled(&tms[i], CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, bufs[i], d, st, bx, es,
                                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
        std::printf("encode failed\n");
        return 1;
      }
    }
    const uint32_t box_bytes = v.bw * 16 * np * 4;
    const uint32_t need = 16 * v.stages * box_bytes;
    const uint32_t sm = v.smem_kb * 1024 > need ? v.smem_kb * 1024 : need;
    CK(cudaFuncSetAttribute(ring_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
    const uint32_t cpw = wpr / v.bw / 4;
    const float us = graph_us(s, 40, [&](int i) {
      P p{v.bw, np, v.stages, cpw, v.delay, v.work, box_bytes, out};
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(rows / 64);
      cfg.blockDim = dim3(512);
      cfg.dynamicSmemBytes = sm;
      cfg.stream = s;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      CK(cudaLaunchKernelEx(&cfg, ring_kernel, tms[i % nbuf], p));
    });
    std::printf("25.2 MB W3 8192^2, 128 CTAs x 16 warps: box {%2u words,16 rows,3 planes} = %5u B, "
                "%u slots/warp, delay %4u, work %4u cyc/item, smem %3u KB: %6.2f us/call %5.0f GB/s\n",
                v.bw, box_bytes, v.stages, v.delay, v.work, sm / 1024, us, bytes / us / 1e3);
  }
  for (auto& b : bufs) cudaFree(b);
  return 0;
}
