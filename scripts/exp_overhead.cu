// Capture-kernel fixed-cost breakdown (experiment, not product code).
// Variants of a 128-bit streaming copy, each adding one piece of the
// capture kernel's protocol, timed as 16 launches replayed in a CUDA graph:
//   0 copy only
//   1 + done counter; last CTA re-arms (no plan)
//   2 + leader election / plan handshake (leader does a dependent chain of
//       L2 reads/writes like tf_reserve), waiters back off up to 2 us
//   3 as 2 with back-off capped at 128 ns
//   4 + last CTA posts a 64-B descriptor to mapped pinned host memory
//   5 as 4, waiters do not wait before the first segment's loads (prefetch)
// build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/exp_overhead scripts/exp_overhead.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

constexpr int kThreads = 256, kWarps = 8, kUnroll = 8, kSeg = 32 * kUnroll;

struct Ctl {
  uint32_t arrive, done, plan_flag, pad;
  uint64_t chain[16];
  uint64_t off;
};

__device__ __forceinline__ uint4 ldnc(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}

template <int V>
__global__ void __launch_bounds__(kThreads, 3) k(const uint4* __restrict__ src, uint4* dst, int64_t words,
                                                 Ctl* c, uint64_t* host_meta, int backoff_cap) {
  __shared__ uint64_t s_off;
  __shared__ uint32_t s_last;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t segs = (words + kSeg - 1) / kSeg;
  const int64_t chunk = (segs + gridDim.x - 1) / gridDim.x;
  const int64_t s0 = blockIdx.x * chunk, s1 = min(s0 + chunk, segs);
  bool leader = false;
  if (V >= 2 && tid == 0) {
    leader = atomicAdd(&c->arrive, 1u) == 0;
    if (leader) {
      uint64_t x = 0;
      for (int i = 0; i < 8; ++i) { x += *(volatile uint64_t*)&c->chain[i]; *(volatile uint64_t*)&c->chain[i] = x + 1; }
      c->off = x & 0;
      __threadfence();
      atomicExch(&c->plan_flag, 1u);
    }
  }
  int64_t s = s0 + warp;
  uint4 v[kUnroll];
  if (V == 5 && s < s1) {
#pragma unroll
    for (int i = 0; i < kUnroll; ++i) {
      int64_t w = s * kSeg + lane + i * 32;
      if (w < words) v[i] = ldnc(src + w);
    }
  }
  if (V >= 2) {
    if (tid == 0) {
      if (!leader) {
        uint32_t ns = 32;
        while (*(volatile uint32_t*)&c->plan_flag == 0) {
          __nanosleep(ns);
          if (V == 2) ns = ns < 2048 ? ns * 2 : ns;
          else ns = ns < (uint32_t)backoff_cap ? ns * 2 : ns;
        }
      }
      s_off = *(volatile uint64_t*)&c->off;
    }
    __syncthreads();
  } else {
    s_off = 0;
  }
  uint4* d = dst + s_off / 16;
  bool have = (V == 5);
  for (; s < s1; s += kWarps) {
    if (!have) {
#pragma unroll
      for (int i = 0; i < kUnroll; ++i) {
        int64_t w = s * kSeg + lane + i * 32;
        if (w < words) v[i] = ldnc(src + w);
      }
    }
    have = false;
#pragma unroll
    for (int i = 0; i < kUnroll; ++i) {
      int64_t w = s * kSeg + lane + i * 32;
      if (w < words) d[w] = v[i];
    }
  }
  if (V >= 1) {
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      s_last = atomicAdd(&c->done, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (s_last) {
      if (V >= 4 && warp == 0 && lane < 8) host_meta[lane] = 0x1234 + lane;
      if (tid == 0) { c->arrive = 0; c->done = 0; c->plan_flag = 0; }
    }
  }
}


// Latency probe: tid 0 of every CTA stamps kernel entry, then the return of
// a dependent chain of loads from a small control block (as the capture
// kernel's prologue does), then a bar.sync; per-CTA stamps go to `out`.
__global__ void __launch_bounds__(kThreads, 3) lat_probe(const uint64_t* ctl, const uint8_t* keep,
                                                          uint64_t* out, const uint4* src, uint4* dst,
                                                          int64_t words) {
  const int tid = threadIdx.x;
  uint64_t t0 = 0, t1 = 0, t2 = 0, t3 = 0;
  __shared__ uint64_t s;
  if (tid == 0) {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    uint64_t v;
    asm volatile("ld.global.cg.u64 %0, [%1];" : "=l"(v) : "l"(ctl + (blockIdx.x % 8) * 16) : "memory");
    s = v;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1) : "l"(v));
    uint64_t w;
    asm volatile("ld.global.cg.u64 %0, [%1];" : "=l"(w) : "l"(ctl + 128 + (v & 1)) : "memory");
    s += w;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t2) : "l"(w));
  }
  uint8_t kb = tid < 8 ? keep[tid] : 0;
  __syncthreads();
  if (tid == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t3) : "l"(s + kb));
  // a little copy so launches overlap like real ones
  int64_t w0 = (int64_t)blockIdx.x * kThreads + tid;
  for (int64_t w = w0; w < words; w += (int64_t)gridDim.x * kThreads) dst[w] = src[w];
  if (tid == 0) {
    out[blockIdx.x * 4 + 0] = t0;
    out[blockIdx.x * 4 + 1] = t1;
    out[blockIdx.x * 4 + 2] = t2;
    out[blockIdx.x * 4 + 3] = t3;
  }
}

void probe_run(int grid, int64_t bytes) {
  uint64_t *ctl, *out;
  uint8_t* keep;
  uint8_t *src, *dst;
  CK(cudaMalloc(&ctl, 4096));
  CK(cudaMemset(ctl, 0, 4096));
  CK(cudaMalloc(&keep, 256));
  CK(cudaMemset(keep, 1, 256));
  CK(cudaMalloc(&out, 16 * 1024 * 4 * 8));
  CK(cudaMalloc(&src, bytes));
  CK(cudaMalloc(&dst, bytes));
  cudaStream_t s;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  const int n = 16;
  cudaGraph_t g;
  cudaGraphExec_t ge;
  CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal));
  for (int i = 0; i < n; ++i)
    lat_probe<<<grid, kThreads, 0, s>>>(ctl, keep, out + (size_t)i * 1024 * 4, (const uint4*)src, (uint4*)dst, bytes / 16);
  CK(cudaStreamEndCapture(s, &g));
  CK(cudaGraphInstantiate(&ge, g, 0));
  for (int r = 0; r < 3; ++r) CK(cudaGraphLaunch(ge, s));
  CK(cudaStreamSynchronize(s));
  std::vector<uint64_t> h((size_t)n * 1024 * 4);
  CK(cudaMemcpy(h.data(), out, h.size() * 8, cudaMemcpyDeviceToHost));
  double a1 = 0, a2 = 0, a3 = 0, m1 = 0, m3 = 0, span = 0;
  for (int i = 1; i < n; ++i) {
    uint64_t e0 = ~0ull, e1 = 0;
    double mx1 = 0, mx3 = 0;
    for (int b = 0; b < grid; ++b) {
      const uint64_t* q = &h[((size_t)i * 1024 + b) * 4];
      e0 = std::min(e0, q[0]);
      a1 += q[1] - q[0]; a2 += q[2] - q[1]; a3 += q[3] - q[0];
      mx1 = std::max(mx1, (double)(q[1] - q[0]));
      mx3 = std::max(mx3, (double)q[3]);
    }
    m1 += mx1;
    m3 += mx3 - e0;
    uint64_t prev0 = ~0ull;
    for (int b = 0; b < grid; ++b) prev0 = std::min(prev0, h[((size_t)(i - 1) * 1024 + b) * 4]);
    span += e0 - prev0;
  }
  double k = (double)(n - 1) * grid;
  printf("probe grid %4d copy %6.1f MiB | ld1 avg %6.0f ns max-avg %6.0f | ld2 (dependent) %6.0f ns | to bar done avg %6.0f ns, latest CTA %6.0f ns | launch-to-launch %6.0f ns\n",
         grid, bytes / 1048576.0, a1 / k, m1 / (n - 1), a2 / k, a3 / k, m3 / (n - 1), span / (n - 1));
}

template <int V>
float run(const uint4* src, uint4* dst, int64_t bytes, Ctl* c, uint64_t* hm, int grid, int cap, int n) {
  cudaStream_t s;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  int64_t words = bytes / 16;
  k<V><<<grid, kThreads, 0, s>>>(src, dst, words, c, hm, cap);
  CK(cudaStreamSynchronize(s));
  cudaGraph_t g;
  cudaGraphExec_t ge;
  CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal));
  for (int i = 0; i < n; ++i) k<V><<<grid, kThreads, 0, s>>>(src, dst, words, c, hm, cap);
  CK(cudaStreamEndCapture(s, &g));
  CK(cudaGraphInstantiate(&ge, g, 0));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  std::vector<float> t;
  for (int r = 0; r < 7; ++r) {
    cudaEventRecord(a, s);
    CK(cudaGraphLaunch(ge, s));
    cudaEventRecord(b, s);
    CK(cudaStreamSynchronize(s));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    t.push_back(ms * 1e3f / n);
  }
  std::sort(t.begin(), t.end());
  cudaGraphExecDestroy(ge);
  cudaGraphDestroy(g);
  cudaStreamDestroy(s);
  return t[t.size() / 2];
}

#include <algorithm>
int main(int argc, char** argv) {
  int64_t sizes[] = {1 << 20, 8 << 20, 32 << 20, 112 << 20};
  uint8_t *src, *dst;
  CK(cudaMalloc(&src, 256 << 20));
  CK(cudaMalloc(&dst, 256 << 20));
  CK(cudaMemset(src, 1, 256 << 20));
  Ctl* c;
  CK(cudaMalloc(&c, sizeof(Ctl)));
  CK(cudaMemset(c, 0, sizeof(Ctl)));
  uint64_t* hm;
  CK(cudaHostAlloc(&hm, 4096, cudaHostAllocMapped));
  uint64_t* hm_dev;
  CK(cudaHostGetDevicePointer((void**)&hm_dev, hm, 0));
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int g : {64, 148, 444}) for (int64_t b : {1 << 20, 8 << 20, 32 << 20}) probe_run(g, b);
  if (argc > 1) return 0;
  const int n = 16;
  for (int64_t bytes : sizes) {
    int grids[] = {sms, 2 * sms, 3 * sms, 4 * sms};
    for (int gm : grids) {
      int grid = (int)std::min<int64_t>(gm, std::max<int64_t>(1, bytes / 16384));
      const uint4* s4 = (const uint4*)src;
      uint4* d4 = (uint4*)dst;
      float t0 = run<0>(s4, d4, bytes, c, hm_dev, grid, 0, n);
      float t1 = run<1>(s4, d4, bytes, c, hm_dev, grid, 128, n);
      float t2 = run<2>(s4, d4, bytes, c, hm_dev, grid, 2048, n);
      float t3 = run<3>(s4, d4, bytes, c, hm_dev, grid, 128, n);
      float t4 = run<4>(s4, d4, bytes, c, hm_dev, grid, 128, n);
      float t5 = run<5>(s4, d4, bytes, c, hm_dev, grid, 128, n);
      printf("bytes %6.1f MiB grid %4d | copy %6.2f | +done %6.2f | +plan(2us) %6.2f | +plan(128ns) %6.2f | +hostdesc %6.2f | +prefetch %6.2f us\n",
             bytes / 1048576.0, grid, t0, t1, t2, t3, t4, t5);
      if (grid < gm) break;
    }
  }
  return 0;
}
