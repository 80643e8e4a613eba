// Microbenchmarks that decide the dense-build (K1) design on B200:
// shared-memory atomic throughput per element type, global RED throughput
// into an L2-resident sketch-sized array, DSMEM remote reductions, and
// L2 / HBM streaming read bandwidth. Run on one GPU; prints one line per test.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA error %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint32_t lcg(uint32_t& s) { s = s * 1664525u + 1013904223u; return s >> 8; }

template <typename T>
__global__ void smem_atomic(T* out, int iters, int mask) {
  extern __shared__ __align__(16) unsigned char sm[];
  T* s = reinterpret_cast<T*>(sm);
  for (int i = threadIdx.x; i <= mask; i += blockDim.x) s[i] = T(0);
  __syncthreads();
  uint32_t st = blockIdx.x * 7919u + threadIdx.x * 104729u;
  T v = T(1);
#pragma unroll 8
  for (int it = 0; it < iters; ++it) atomicAdd(&s[lcg(st) & mask], v);
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = s[blockIdx.x & mask];
}

// Non-atomic racy read-modify-write: the ceiling for a conflict-free scheme.
__global__ void smem_racy_f64(double* out, int iters, int mask) {
  extern __shared__ __align__(16) unsigned char sm[];
  double* s = reinterpret_cast<double*>(sm);
  for (int i = threadIdx.x; i <= mask; i += blockDim.x) s[i] = 0;
  __syncthreads();
  uint32_t st = blockIdx.x * 7919u + threadIdx.x * 104729u;
#pragma unroll 8
  for (int it = 0; it < iters; ++it) { volatile double* p = &s[lcg(st) & mask]; *p = *p + 1.0; }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = s[blockIdx.x & mask];
}

// Two-limb int32 fixed point: two native ATOMS.ADD per contribution.
__global__ void smem_2limb(unsigned* out, int iters, int mask) {
  extern __shared__ __align__(16) unsigned char sm[];
  unsigned* s = reinterpret_cast<unsigned*>(sm);
  for (int i = threadIdx.x; i <= 2 * mask + 1; i += blockDim.x) s[i] = 0;
  __syncthreads();
  uint32_t st = blockIdx.x * 7919u + threadIdx.x * 104729u;
#pragma unroll 8
  for (int it = 0; it < iters; ++it) {
    uint32_t a = lcg(st) & mask;
    atomicAdd(&s[a], 3u);
    atomicAdd(&s[mask + 1 + a], 5u);
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = s[blockIdx.x & mask];
}

template <typename T>
__global__ void gmem_red(T* arr, int iters, int mask) {
  uint32_t st = blockIdx.x * 7919u + threadIdx.x * 104729u;
  T v = T(1);
#pragma unroll 8
  for (int it = 0; it < iters; ++it) atomicAdd(&arr[lcg(st) & mask], v);
}

__global__ void __cluster_dims__(2, 1, 1) dsmem_red(double* out, int iters, int mask) {
  extern __shared__ __align__(16) unsigned char sm[];
  double* s = reinterpret_cast<double*>(sm);
  cg::cluster_group cl = cg::this_cluster();
  for (int i = threadIdx.x; i <= mask; i += blockDim.x) s[i] = 0;
  cl.sync();
  double* remote = cl.map_shared_rank(s, cl.block_rank() ^ 1);
  uint32_t st = blockIdx.x * 7919u + threadIdx.x * 104729u;
#pragma unroll 8
  for (int it = 0; it < iters; ++it) atomicAdd(&remote[lcg(st) & mask], 1.0);
  cl.sync();
  if (threadIdx.x == 0) out[blockIdx.x] = s[blockIdx.x & mask];
}

__global__ void stream_read(const double2* __restrict__ a, size_t n, int passes, double* out) {
  double acc = 0;
  for (int p = 0; p < passes; ++p)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
      double2 v = __ldcg(&a[i]);
      acc += v.x + v.y;
    }
  if (acc == 123.456) out[0] = acc;
}

template <typename K>
float time_it(K launch, int reps = 5) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  launch(); cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"sms\": %d, \"clock_khz\": %d}\n", sms, clk);
  void* buf; CK(cudaMalloc(&buf, 1 << 20));
  const int threads = 512, iters = 4096;
  for (int cps : {1, 2, 4}) {
    int grid = sms * cps;
    size_t smem_bytes = (cps == 1) ? (160 << 10) : (cps == 2 ? (96 << 10) : (48 << 10));
    double ops = (double)grid * threads * iters;
#define RUN_SMEM(KERN, T, NAME, ELEMS)                                                                  \
    {                                                                                                 \
      int mask = (int)(ELEMS) - 1;                                                                    \
      CK(cudaFuncSetAttribute(KERN, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes));   \
      float ms = time_it([&] { KERN<<<grid, threads, smem_bytes>>>((T*)buf, iters, mask); });          \
      CK(cudaGetLastError());                                                                         \
      printf("{\"test\": \"%s\", \"ctas_per_sm\": %d, \"elems\": %d, \"ms\": %.4f, \"Gops\": %.1f, \"ops_per_clk_per_sm\": %.3f}\n", \
             NAME, cps, mask + 1, ms, ops / ms / 1e6, ops / (ms * 1e-3) / sms / (clk * 1e3));         \
    }
    size_t pow2 = 1; while (pow2 * 2 * 8 <= smem_bytes) pow2 *= 2;   // elements for 8-byte types
    RUN_SMEM(smem_atomic<unsigned>, unsigned, "smem_u32_atomsadd", pow2 * 2)
    RUN_SMEM(smem_atomic<float>, float, "smem_f32_cas", pow2 * 2)
    RUN_SMEM(smem_atomic<double>, double, "smem_f64_cas", pow2)
    RUN_SMEM(smem_atomic<unsigned long long>, unsigned long long, "smem_u64_cas", pow2)
    RUN_SMEM(smem_racy_f64, double, "smem_f64_racy_rmw", pow2)
    RUN_SMEM(smem_2limb, unsigned, "smem_2limb_u32_pairs", pow2)
  }
  // global RED into sketch-sized (L2 resident) arrays
  void* garr; CK(cudaMalloc(&garr, 64ull << 20));
  for (int mb : {1, 5, 40}) {
    int grid = sms * 8, th = 256;
    double ops = (double)grid * th * iters;
    int mask8 = (int)((size_t(mb) << 20) / 8) - 1;
    int mask4 = (int)((size_t(mb) << 20) / 4) - 1;
    float ms = time_it([&] { gmem_red<double><<<grid, th>>>((double*)garr, iters, mask8); });
    printf("{\"test\": \"gmem_red_f64\", \"MB\": %d, \"ms\": %.4f, \"Gops\": %.1f}\n", mb, ms, ops / ms / 1e6);
    ms = time_it([&] { gmem_red<float><<<grid, th>>>((float*)garr, iters, mask4); });
    printf("{\"test\": \"gmem_red_f32\", \"MB\": %d, \"ms\": %.4f, \"Gops\": %.1f}\n", mb, ms, ops / ms / 1e6);
    ms = time_it([&] { gmem_red<unsigned long long><<<grid, th>>>((unsigned long long*)garr, iters, mask8); });
    printf("{\"test\": \"gmem_red_u64\", \"MB\": %d, \"ms\": %.4f, \"Gops\": %.1f}\n", mb, ms, ops / ms / 1e6);
  }
  {
    int grid = (sms / 2) * 2, th = 512;
    size_t smem_bytes = 96 << 10;
    CK(cudaFuncSetAttribute(dsmem_red, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes));
    double ops = (double)grid * th * iters;
    float ms = time_it([&] { dsmem_red<<<grid, th, smem_bytes>>>((double*)buf, iters, 8191); });
    CK(cudaGetLastError());
    printf("{\"test\": \"dsmem_red_f64_cluster2\", \"ms\": %.4f, \"Gops\": %.1f}\n", ms, ops / ms / 1e6);
  }
  // streaming read bandwidth: L2-resident (64 MB) and HBM (4 GB)
  for (size_t mb : {32ull, 64ull, 4096ull}) {
    void* a; CK(cudaMalloc(&a, mb << 20)); CK(cudaMemset(a, 0, mb << 20));
    size_t n = (mb << 20) / 16;
    int passes = mb <= 64 ? 20 : 1;
    for (int cps : {4, 8}) {
      float ms = time_it([&] { stream_read<<<sms * cps, 512>>>((const double2*)a, n, passes, (double*)buf); });
      printf("{\"test\": \"stream_read\", \"MB\": %zu, \"ctas_per_sm\": %d, \"ms\": %.4f, \"GBps\": %.1f}\n",
             mb, cps, ms, (double)(mb << 20) * passes / ms / 1e6);
    }
    cudaFree(a);
  }
  return 0;
}
