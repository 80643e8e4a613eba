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


// Conflict structure of u32 ATOMS: lane L hits bank (L * stride) mod 32 of a random
// 32-word row, so stride 1 is conflict-free, 2 gives 2-way, 32 gives 32-way conflicts;
// stride 0 keeps fully random banks (the reference point above).
__global__ void smem_u32_banks(unsigned* out, int iters, int mask, int stride) {
  extern __shared__ __align__(16) unsigned char sm[];
  unsigned* s = reinterpret_cast<unsigned*>(sm);
  for (int i = threadIdx.x; i <= mask; i += blockDim.x) s[i] = 0;
  __syncthreads();
  const unsigned lane = threadIdx.x & 31;
  uint32_t st = blockIdx.x * 7919u + (threadIdx.x >> 5) * 104729u;  // warp-uniform row stream
#pragma unroll 8
  for (int it = 0; it < iters; ++it) {
    const uint32_t r = lcg(st);
    const uint32_t a = stride ? (((r << 5) + lane * stride) & mask) : ((r * 2654435761u + lane * 40503u) & mask);
    atomicAdd(&s[a], 1u);
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = s[blockIdx.x & mask];
}

// Exact 64-bit add as two limbs, the build kernel's pattern: ATOMS.ADD with return on the
// low limb, the carry into a RED on the high limb (conflict-free or random banks).
__global__ void smem_2limb_ret(unsigned* out, int iters, int mask, int cf) {
  extern __shared__ __align__(16) unsigned char sm[];
  unsigned* s = reinterpret_cast<unsigned*>(sm);
  for (int i = threadIdx.x; i <= 2 * mask + 1; i += blockDim.x) s[i] = 0;
  __syncthreads();
  const unsigned lane = threadIdx.x & 31;
  uint32_t st = blockIdx.x * 7919u + (threadIdx.x >> 5) * 104729u + (cf ? 0u : lane * 7u);
  uint32_t v = 0x9e3779b9u * (threadIdx.x + 1);
#pragma unroll 4
  for (int it = 0; it < iters; ++it) {
    const uint32_t r = lcg(st);
    const uint32_t a = cf ? (((r << 5) + lane) & mask) : (r & mask);
    v = v * 1664525u + 1013904223u;
    const unsigned old = atomicAdd(&s[a], v);
    const unsigned c = (old + v) < old;
    atomicAdd(&s[mask + 1 + a], (v >> 28) + c);
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = s[blockIdx.x & mask];
}

// One limb with the rare carry: |q| < 2^qb, the high limb (global, RED) is touched only
// when the low limb wraps (probability ~|q| / 2^32 per add).
__global__ void smem_1limb_rare(unsigned* out, unsigned long long* hi, int iters, int mask, int cf, int qb) {
  extern __shared__ __align__(16) unsigned char sm[];
  unsigned* s = reinterpret_cast<unsigned*>(sm);
  for (int i = threadIdx.x; i <= mask; i += blockDim.x) s[i] = 0;
  __syncthreads();
  const unsigned lane = threadIdx.x & 31;
  uint32_t st = blockIdx.x * 7919u + (threadIdx.x >> 5) * 104729u + (cf ? 0u : lane * 7u);
  uint32_t v = 0x9e3779b9u * (threadIdx.x + 1);
  const int sh = 32 - qb;
#pragma unroll 4
  for (int it = 0; it < iters; ++it) {
    const uint32_t r = lcg(st);
    const uint32_t a = cf ? (((r << 5) + lane) & mask) : (r & mask);
    v = v * 1664525u + 1013904223u;
    const int q = static_cast<int>(v) >> sh;  // signed, |q| < 2^(qb-1)
    const unsigned old = atomicAdd(&s[a], static_cast<unsigned>(q));
    const unsigned nw = old + static_cast<unsigned>(q);
    const int d = q >= 0 ? (nw < old ? 1 : 0) : (nw > old ? -1 : 0);
    if (d) atomicAdd(hi + ((blockIdx.x * 4096u + a) & ((1u << 22) - 1)), static_cast<unsigned long long>(static_cast<long long>(d)));
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = s[blockIdx.x & mask];
}

// Native u32 reduction into the partner CTA's shared memory (cluster of 2).
__global__ void __cluster_dims__(2, 1, 1) dsmem_red_u32(unsigned* out, int iters, int mask, int cf) {
  extern __shared__ __align__(16) unsigned char sm[];
  unsigned* s = reinterpret_cast<unsigned*>(sm);
  cg::cluster_group cl = cg::this_cluster();
  for (int i = threadIdx.x; i <= mask; i += blockDim.x) s[i] = 0;
  cl.sync();
  unsigned* remote = cl.map_shared_rank(s, cl.block_rank() ^ 1);
  const unsigned lane = threadIdx.x & 31;
  uint32_t st = blockIdx.x * 7919u + (threadIdx.x >> 5) * 104729u + (cf ? 0u : lane * 7u);
#pragma unroll 8
  for (int it = 0; it < iters; ++it) {
    const uint32_t r = lcg(st);
    const uint32_t a = cf ? (((r << 5) + lane) & mask) : (r & mask);
    atomicAdd(&remote[a], 1u);
  }
  cl.sync();
  if (threadIdx.x == 0) out[blockIdx.x] = s[blockIdx.x & mask];
}

// Shared-memory reads: 4- or 8-byte words at random or conflict-free addresses.
template <typename T>
__global__ void smem_read(unsigned* out, int iters, int mask, int cf) {
  extern __shared__ __align__(16) unsigned char sm[];
  T* s = reinterpret_cast<T*>(sm);
  for (int i = threadIdx.x; i <= mask; i += blockDim.x) s[i] = T(i);
  __syncthreads();
  const unsigned lane = threadIdx.x & 31;
  uint32_t st = blockIdx.x * 7919u + (threadIdx.x >> 5) * 104729u + (cf ? 0u : lane * 7u);
  T acc = T(0);
#pragma unroll 8
  for (int it = 0; it < iters; ++it) {
    const uint32_t r = lcg(st);
    const uint32_t a = cf ? (((r << 5) + lane) & mask) : (r & mask);
    acc += s[a];
  }
  if (acc == T(12345)) out[blockIdx.x] = (unsigned)acc;
}

// L2 gathers of 4-byte words from an L2-resident array: each lane of a warp reads one
// word from its own random 32-byte sector (stride 0), or the warp reads words spaced
// `stride` apart inside one random row (the class-list gather pattern).
__global__ void l2_gather(const float* __restrict__ a, int iters, unsigned mask, int stride, float* out) {
  const unsigned lane = threadIdx.x & 31;
  uint32_t st = blockIdx.x * 7919u + (threadIdx.x >> 5) * 104729u + (stride ? 0u : lane * 7u);
  float acc = 0;
#pragma unroll 8
  for (int it = 0; it < iters; ++it) {
    const uint32_t r = lcg(st);
    const uint32_t idx = stride ? (((r << 10) + lane * stride) & mask) : ((r << 3) & mask);
    acc += __ldg(a + idx);
  }
  if (acc == 123.456f) out[0] = acc;
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
  // ---- round 2: bank structure of the scatter (one CTA of 1024 threads per SM, 128 KB) ----
  {
    const int th = 1024, it2 = 2048, grid = sms;
    const size_t sb = 128 << 10;
    const int mask = (int)(sb / 4) - 1;
    double ops = (double)grid * th * it2;
    CK(cudaFuncSetAttribute(smem_u32_banks, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sb));
    for (int stride : {0, 1, 2, 4, 8, 32}) {
      float ms = time_it([&] { smem_u32_banks<<<grid, th, sb>>>((unsigned*)buf, it2, mask, stride); });
      CK(cudaGetLastError());
      printf("{\"test\": \"smem_u32_atoms_banks\", \"lane_stride\": %d, \"ms\": %.4f, \"ops_per_clk_per_sm\": %.3f}\n",
             stride, ms, ops / (ms * 1e-3) / sms / (clk * 1e3));
    }
    CK(cudaFuncSetAttribute(smem_2limb_ret, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sb));
    for (int cf : {0, 1}) {
      float ms = time_it([&] { smem_2limb_ret<<<grid, th, sb>>>((unsigned*)buf, it2, mask / 2, cf); });
      CK(cudaGetLastError());
      printf("{\"test\": \"smem_2limb_carry\", \"conflict_free\": %d, \"ms\": %.4f, \"adds_per_clk_per_sm\": %.3f}\n",
             cf, ms, ops / (ms * 1e-3) / sms / (clk * 1e3));
    }
    unsigned long long* hi; CK(cudaMalloc(&hi, 8ull << 22)); CK(cudaMemset(hi, 0, 8ull << 22));
    CK(cudaFuncSetAttribute(smem_1limb_rare, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sb));
    for (int qb : {24, 28}) for (int cf : {0, 1}) {
      float ms = time_it([&] { smem_1limb_rare<<<grid, th, sb>>>((unsigned*)buf, hi, it2, mask, cf, qb); });
      CK(cudaGetLastError());
      printf("{\"test\": \"smem_1limb_rare_carry\", \"q_bits\": %d, \"conflict_free\": %d, \"ms\": %.4f, \"adds_per_clk_per_sm\": %.3f}\n",
             qb, cf, ms, ops / (ms * 1e-3) / sms / (clk * 1e3));
    }
    CK(cudaFuncSetAttribute(dsmem_red_u32, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sb));
    for (int cf : {0, 1}) {
      float ms = time_it([&] { dsmem_red_u32<<<(grid / 2) * 2, th, sb>>>((unsigned*)buf, it2, mask, cf); });
      CK(cudaGetLastError());
      printf("{\"test\": \"dsmem_red_u32_cluster2\", \"conflict_free\": %d, \"ms\": %.4f, \"ops_per_clk_per_sm\": %.3f}\n",
             cf, ms, (double)((grid / 2) * 2) * th * it2 / (ms * 1e-3) / sms / (clk * 1e3));
    }
    CK(cudaFuncSetAttribute(smem_read<unsigned>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sb));
    CK(cudaFuncSetAttribute(smem_read<unsigned long long>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sb));
    for (int cf : {0, 1}) {
      float ms = time_it([&] { smem_read<unsigned><<<grid, th, sb>>>((unsigned*)buf, it2, mask, cf); });
      printf("{\"test\": \"smem_read_u32\", \"conflict_free\": %d, \"ms\": %.4f, \"ops_per_clk_per_sm\": %.3f}\n",
             cf, ms, ops / (ms * 1e-3) / sms / (clk * 1e3));
      ms = time_it([&] { smem_read<unsigned long long><<<grid, th, sb>>>((unsigned*)buf, it2, mask / 2, cf); });
      printf("{\"test\": \"smem_read_u64\", \"conflict_free\": %d, \"ms\": %.4f, \"ops_per_clk_per_sm\": %.3f}\n",
             cf, ms, ops / (ms * 1e-3) / sms / (clk * 1e3));
    }
    float* g; CK(cudaMalloc(&g, 64ull << 20)); CK(cudaMemset(g, 0, 64ull << 20));
    for (int stride : {0, 1, 2, 4, 8}) {
      float ms = time_it([&] { l2_gather<<<grid * 2, 512>>>(g, it2, (16u << 20) - 1, stride, (float*)buf); });
      double loads = (double)grid * 2 * 512 * it2;
      printf("{\"test\": \"l2_gather_f32\", \"lane_stride\": %d, \"ms\": %.4f, \"Gloads\": %.1f, \"useful_GBps\": %.1f}\n",
             stride, ms, loads / ms / 1e6, loads * 4 / ms / 1e6);
    }
  }
  return 0;
}
