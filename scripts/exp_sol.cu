// Speed-of-light reference for the capture kernel (experiment, not product
// code): how fast can ANY kernel copy the same bytes, launched the way the
// capture kernel is (back to back in a CUDA graph, with and without PDL)?
//
//   sol    grid-stride 128-bit copy, 256 threads, 8 words in flight per
//          thread, grid = 148 x k CTAs
//   memcpy cudaMemcpyAsync D2D of the same bytes
//
// Sources and destinations rotate over 4 buffers each so large copies are
// not L2 hits (decode-size copies are, as in a model where the producer
// kernel just wrote them).
// build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/exp_sol scripts/exp_sol.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                       \
  do {                                                                              \
    cudaError_t e = (x);                                                            \
    if (e != cudaSuccess) {                                                         \
      printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e));              \
      exit(1);                                                                      \
    }                                                                               \
  } while (0)

__device__ __forceinline__ uint4 ldnc(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

template <int U>
__global__ void __launch_bounds__(256) sol(const uint4* __restrict__ src, uint4* __restrict__ dst,
                                           int64_t words) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < words; i += U * stride) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = ldnc(src + i + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) dst[i + u * stride] = v[u];
  }
  for (; i < words; i += stride) dst[i] = ldnc(src + i);
}

static float time_graph(cudaGraphExec_t ge, cudaStream_t s, int reps, int n) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  std::vector<float> t;
  for (int r = 0; r < reps; ++r) {
    CK(cudaEventRecord(a, s));
    CK(cudaGraphLaunch(ge, s));
    CK(cudaEventRecord(b, s));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    t.push_back(ms * 1e3f / n);
  }
  std::sort(t.begin(), t.end());
  return t[t.size() / 2];
}

int main(int argc, char** argv) {
  const int n = 16, reps = 7;
  std::vector<size_t> sizes = {128u << 10, 448u << 10, 512u << 10, 1792u << 10, 1u << 20,
                               8u << 20,   32u << 20,  112u << 20};
  size_t maxb = 112u << 20;
  uint8_t *src[4], *dst[4];
  for (int i = 0; i < 4; ++i) {
    CK(cudaMalloc(&src[i], maxb));
    CK(cudaMalloc(&dst[i], maxb));
    CK(cudaMemset(src[i], i + 1, maxb));
  }
  cudaStream_t s;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  int grids[] = {148, 296, 444, 592};
  if (argc > 1) sizes.clear();  // ncu mode: only the three single launches below
  for (size_t bytes : sizes) {
    const int64_t words = bytes / 16;
    for (int pdl = 0; pdl < 2; ++pdl) {
      for (int g : grids) {
        cudaGraph_t gr;
        CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal));
        for (int k = 0; k < n; ++k) {
          cudaLaunchConfig_t cfg = {};
          cfg.gridDim = dim3(std::max<int64_t>(1, std::min<int64_t>(g, (words + 255) / 256)));
          cfg.blockDim = dim3(256);
          cfg.stream = s;
          cudaLaunchAttribute at[1];
          at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
          at[0].val.programmaticStreamSerializationAllowed = 1;
          cfg.attrs = at;
          cfg.numAttrs = pdl;
          CK(cudaLaunchKernelEx(&cfg, sol<8>, (const uint4*)src[k % 4], (uint4*)dst[k % 4], words));
        }
        CK(cudaStreamEndCapture(s, &gr));
        cudaGraphExec_t ge;
        CK(cudaGraphInstantiate(&ge, gr, 0));
        CK(cudaGraphLaunch(ge, s));
        CK(cudaStreamSynchronize(s));
        float us = time_graph(ge, s, reps, n);
        printf("{\"kind\": \"sol\", \"bytes\": %zu, \"grid\": %d, \"pdl\": %d, \"us\": %.3f, \"gbs_rw\": %.1f}\n",
               bytes, g, pdl, us, 2.0 * bytes / (us * 1e3));
        CK(cudaGraphExecDestroy(ge));
        CK(cudaGraphDestroy(gr));
      }
    }
    {
      cudaGraph_t gr;
      CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal));
      for (int k = 0; k < n; ++k)
        CK(cudaMemcpyAsync(dst[k % 4], src[k % 4], bytes, cudaMemcpyDeviceToDevice, s));
      CK(cudaStreamEndCapture(s, &gr));
      cudaGraphExec_t ge;
      CK(cudaGraphInstantiate(&ge, gr, 0));
      CK(cudaGraphLaunch(ge, s));
      CK(cudaStreamSynchronize(s));
      float us = time_graph(ge, s, reps, n);
      printf("{\"kind\": \"memcpy\", \"bytes\": %zu, \"us\": %.3f, \"gbs_rw\": %.1f}\n", bytes, us,
             2.0 * bytes / (us * 1e3));
      CK(cudaGraphExecDestroy(ge));
      CK(cudaGraphDestroy(gr));
    }
    fflush(stdout);
  }
  // one launch of each at 32 MiB for ncu (grid 296, PDL off)
  if (argc > 1) {
    sol<8><<<296, 256, 0, s>>>((const uint4*)src[0], (uint4*)dst[0], (32 << 20) / 16);
    CK(cudaMemcpyAsync(dst[1], src[1], 32 << 20, cudaMemcpyDeviceToDevice, s));
    sol<8><<<296, 256, 0, s>>>((const uint4*)src[2], (uint4*)dst[2], (112 << 20) / 16);
    CK(cudaStreamSynchronize(s));
  }
  return 0;
}
