// Measured ceilings for the FP64 local-FFT kernels (contraction, moment, LDA) on one B200:
// the DFMA issue rate (independent chains, full occupancy) and the shared-memory bandwidth
// for the 16-byte complex elements those kernels move (conflict-free LDS.128 / STS.128).
// Prints one JSON line per test; bench.py reads the committed copy under profiles/ for the
// contraction's FP64 fraction (the vendor figure is not used).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA error %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

// 8 independent fma chains per thread
__global__ void __launch_bounds__(256) dfma_peak(double* out, int iters, double a, double b) {
  double v[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) v[q] = threadIdx.x * 1e-3 + q;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int q = 0; q < 8; ++q) v[q] = fma(v[q], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int q = 0; q < 8; ++q) s += v[q];
  if (s == 123.456) out[0] = s;
}

// conflict-free 16-byte shared-memory loads (and stores): lane l touches element base + l
template <bool STORE>
__global__ void __launch_bounds__(256) smem_vec16(double* out, int iters, int elems) {
  extern __shared__ __align__(16) double2 s16[];
  for (int i = threadIdx.x; i < elems; i += blockDim.x) s16[i] = make_double2(i, -i);
  __syncthreads();
  double2 acc = make_double2(0.0, 0.0);
  int p = threadIdx.x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (STORE) {
        s16[p] = acc;
        acc.x += 1.0;
      } else {
        const double2 t = s16[p];
        acc.x += t.x;
        acc.y += t.y;
      }
      p += 256;
      if (p >= elems) p -= elems;
    }
  }
  __syncthreads();
  if (acc.x + acc.y + s16[threadIdx.x].x == 123.456) out[0] = acc.x;
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
  double* buf; CK(cudaMalloc(&buf, 1 << 20));
  for (int cps : {2, 4, 8}) {
    const int iters = 4096, grid = sms * cps;
    float ms = time_it([&] { dfma_peak<<<grid, 256>>>(buf, iters, 0.999999, 1e-9); });
    CK(cudaGetLastError());
    const double fmas = (double)grid * 256 * iters * 32;
    printf("{\"test\": \"dfma_peak\", \"ctas_per_sm\": %d, \"ms\": %.4f, \"tflops\": %.2f, \"fma_per_clk_per_sm\": %.2f}\n",
           cps, ms, 2.0 * fmas / ms / 1e9, fmas / (ms * 1e-3) / sms / (clk * 1e3));
  }
  for (int cps : {1, 2, 3}) {
    const int iters = 2048, grid = sms * cps, elems = 4096;  // 64 KB per CTA
    const size_t sb = (size_t)elems * 16;
    CK(cudaFuncSetAttribute(smem_vec16<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sb));
    CK(cudaFuncSetAttribute(smem_vec16<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sb));
    const double bytes = (double)grid * 256 * iters * 8 * 16;
    float ms = time_it([&] { smem_vec16<false><<<grid, 256, sb>>>(buf, iters, elems); });
    CK(cudaGetLastError());
    printf("{\"test\": \"smem_lds128\", \"ctas_per_sm\": %d, \"ms\": %.4f, \"TBps\": %.2f, \"bytes_per_clk_per_sm\": %.1f}\n", cps, ms,
           bytes / ms / 1e9, bytes / (ms * 1e-3) / sms / (clk * 1e3));
    ms = time_it([&] { smem_vec16<true><<<grid, 256, sb>>>(buf, iters, elems); });
    CK(cudaGetLastError());
    printf("{\"test\": \"smem_sts128\", \"ctas_per_sm\": %d, \"ms\": %.4f, \"TBps\": %.2f, \"bytes_per_clk_per_sm\": %.1f}\n", cps, ms,
           bytes / ms / 1e9, bytes / (ms * 1e-3) / sms / (clk * 1e3));
  }
  return 0;
}
