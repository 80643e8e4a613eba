// LDA parameter recovery and held-out likelihood on the device (lda.cpp:228-320).
//
//   recover_params: mu_i = 0.5 (alpha0 + 2) lambda_i unwhiten A[:, i] (one V x k x k product)
//     and Phi[:, i] = the Euclidean projection of mu_i onto the probability simplex
//     (lda.cpp:250-271). The reference sorts the V values and scans the prefix sums for
//     the threshold theta; here one CTA per component finds theta by bisection on
//     f(theta) = sum max(y - theta, 0) = 1 and then recomputes it exactly from the support
//     {y > theta} as (sum - 1) / |support| -- the same threshold (an element at the
//     boundary contributes 0 either way), summed in index order instead of sorted order.
//   heldout_likelihood: per held-out document, 500 projected-gradient steps on the mixture
//     pi (step 1 / largest eigenvalue of the k x k Gram, stop at |step| <= 1e-8), then the
//     mean log-likelihood per token with word probabilities floored at 1e-12. One warp per
//     document, the Gram in shared memory, the k mixture weights spread over the lanes; the
//     k-point simplex projection inside each step is the same bisection at warp scope.
#include <cuda_runtime.h>

#include <cmath>

#include "skc_internal.hpp"

namespace skc {

namespace {

template <int NT>
__device__ double block_reduce_sum(double v, double* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    double t = 0.0;
    for (int w = 0; w < NT / 32; ++w) t += red[w];  // fixed order, every thread
    __syncthreads();
    return t;
}
template <int NT>
__device__ double block_reduce_max(double v, double* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    double t = -INFINITY;
    for (int w = 0; w < NT / 32; ++w) t = fmax(t, red[w]);
    __syncthreads();
    return t;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

}  // namespace

// mu[i][w] = 0.5 (alpha0 + 2) lambda_i sum_c unwhiten[w][c] A[c][i]   (A k x k row-major)
__global__ void __launch_bounds__(256) k_recover_mu(int V, int k, const double* __restrict__ lambda,
                                                   const double* __restrict__ A, const double* __restrict__ unwhiten,
                                                   double alpha0, double* __restrict__ mu) {
    extern __shared__ double acol[];  // A[:, i]
    const int i = blockIdx.y;
    for (int c = threadIdx.x; c < k; c += blockDim.x) acol[c] = A[static_cast<size_t>(c) * k + i];
    __syncthreads();
    const int w = blockIdx.x * blockDim.x + threadIdx.x;
    if (w >= V) return;
    const double* u = unwhiten + static_cast<size_t>(w) * k;
    double s = 0.0;
    for (int c = 0; c < k; ++c) s += u[c] * acol[c];
    mu[static_cast<size_t>(i) * V + w] = 0.5 * (alpha0 + 2.0) * lambda[i] * s;
}

// Phi[w][i] = max(mu[i][w] - theta_i, 0), theta_i the simplex threshold of row i.
template <int NT>
__global__ void __launch_bounds__(NT) k_simplex_rows(int V, int k, const double* __restrict__ mu,
                                                     double* __restrict__ Phi) {
    __shared__ double red[NT / 32];
    const int i = blockIdx.x;
    const double* y = mu + static_cast<size_t>(i) * V;
    double mx = -INFINITY;
    for (int w = threadIdx.x; w < V; w += NT) mx = fmax(mx, y[w]);
    mx = block_reduce_max<NT>(mx, red);
    // f(theta) = sum max(y - theta, 0) is decreasing; f(max - 1) >= 1 > f(max) = 0
    double lo = mx - 1.0, hi = mx;
    for (int it = 0; it < 100 && hi - lo > 0.0; ++it) {
        const double mid = 0.5 * (lo + hi);
        if (mid <= lo || mid >= hi) break;
        double f = 0.0;
        for (int w = threadIdx.x; w < V; w += NT) f += fmax(y[w] - mid, 0.0);
        f = block_reduce_sum<NT>(f, red);
        if (f >= 1.0) lo = mid;
        else hi = mid;
    }
    double s = 0.0, cnt = 0.0;
    for (int w = threadIdx.x; w < V; w += NT)
        if (y[w] > lo) {
            s += y[w];
            cnt += 1.0;
        }
    s = block_reduce_sum<NT>(s, red);
    cnt = block_reduce_sum<NT>(cnt, red);
    const bool collapsed = !(cnt > 0.0) || !isfinite(s);  // lda.cpp:262-265 fallback
    const double theta = collapsed ? 0.0 : (s - 1.0) / cnt;
    for (int w = threadIdx.x; w < V; w += NT)
        Phi[static_cast<size_t>(w) * k + i] = collapsed ? 1.0 / V : fmax(y[w] - theta, 0.0);
}

void launch_lda_recover_params(cudaStream_t st, int V, int k, const double* lambda, const double* A,
                               const double* unwhiten, double alpha0, double* mu, double* Phi) {
    dim3 g((V + 255) / 256, k);
    k_recover_mu<<<g, 256, sizeof(double) * k, st>>>(V, k, lambda, A, unwhiten, alpha0, mu);
    count_launch();
    k_simplex_rows<1024><<<k, 1024, 0, st>>>(V, k, mu, Phi);
    count_launch();
}

// Gram G[a][b] = sum_w Phi[w][a] Phi[w][b]: one block per a, threads over b, w in order.
__global__ void k_phi_gram(int V, int k, const double* __restrict__ Phi, double* __restrict__ G) {
    const int a = blockIdx.x;
    for (int b = threadIdx.x; b < k; b += blockDim.x) {
        double s = 0.0;
        for (int w = 0; w < V; ++w) s += Phi[static_cast<size_t>(w) * k + a] * Phi[static_cast<size_t>(w) * k + b];
        G[static_cast<size_t>(b) * k + a] = s;
    }
}
void launch_phi_gram(cudaStream_t st, int V, int k, const double* Phi, double* G) {
    k_phi_gram<<<k, std::min(1024, (k + 31) / 32 * 32), 0, st>>>(V, k, Phi, G);
    count_launch();
}

// k-point simplex projection of x (lane l holds x[l + 32 j], j < KJ), warp scope.
template <int KJ>
__device__ __forceinline__ void warp_simplex(double (&x)[KJ], int k) {
    const int lane = threadIdx.x & 31;
    double mx = -INFINITY;
#pragma unroll
    for (int j = 0; j < KJ; ++j)
        if (lane + 32 * j < k) mx = fmax(mx, x[j]);
    mx = warp_max(mx);
    double lo = mx - 1.0, hi = mx;
    for (int it = 0; it < 100; ++it) {
        const double mid = 0.5 * (lo + hi);
        if (mid <= lo || mid >= hi) break;
        double f = 0.0;
#pragma unroll
        for (int j = 0; j < KJ; ++j)
            if (lane + 32 * j < k) f += fmax(x[j] - mid, 0.0);
        f = warp_sum(f);
        if (f >= 1.0) lo = mid;
        else hi = mid;
    }
    double s = 0.0, c = 0.0;
#pragma unroll
    for (int j = 0; j < KJ; ++j)
        if (lane + 32 * j < k && x[j] > lo) {
            s += x[j];
            c += 1.0;
        }
    s = warp_sum(s);
    c = warp_sum(c);
    const bool collapsed = !(c > 0.0) || !isfinite(s);
    const double theta = collapsed ? 0.0 : (s - 1.0) / c;
#pragma unroll
    for (int j = 0; j < KJ; ++j) x[j] = collapsed ? 1.0 / k : fmax(x[j] - theta, 0.0);
}

// One warp per held-out document: per[d] = mean log-likelihood per token (or NaN if unused),
// floored[d] = words whose probability was floored.
template <int KJ>
__global__ void __launch_bounds__(256) k_heldout_docs(int k, long long D, const long long* __restrict__ doc_ptr,
                                                      const int* __restrict__ word, const int* __restrict__ count,
                                                      const double* __restrict__ Phi, const double* __restrict__ Gg,
                                                      double step, double* __restrict__ per,
                                                      long long* __restrict__ floored) {
    extern __shared__ double G[];  // k x k (column b at G[b*k + a]), then 8 warps x k pi
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int x = threadIdx.x; x < k * k; x += blockDim.x) G[x] = Gg[x];
    __syncthreads();
    double* pis = G + static_cast<size_t>(k) * k + static_cast<size_t>(warp) * k;
    for (long long d = static_cast<long long>(blockIdx.x) * 8 + warp; d < D; d += static_cast<long long>(gridDim.x) * 8) {
        const long long q0 = doc_ptr[d], q1 = doc_ptr[d + 1];
        long long tot = 0;
        for (long long q = q0 + lane; q < q1; q += 32) tot += count[q];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
        if (tot < 1) {
            if (lane == 0) {
                per[d] = NAN;
                floored[d] = 0;
            }
            continue;
        }
        double pi[KJ], phi_tw[KJ];
#pragma unroll
        for (int j = 0; j < KJ; ++j) {
            pi[j] = 1.0 / k;
            phi_tw[j] = 0.0;
        }
        if (k > 1) {
            const double inv_m = 1.0 / static_cast<double>(tot);
            for (long long q = q0; q < q1; ++q) {
                const double c = inv_m * count[q];
                const double* row = Phi + static_cast<size_t>(word[q]) * k;
#pragma unroll
                for (int j = 0; j < KJ; ++j)
                    if (lane + 32 * j < k) phi_tw[j] += c * row[lane + 32 * j];
            }
            for (int it = 0; it < 500; ++it) {
#pragma unroll
                for (int j = 0; j < KJ; ++j)
                    if (lane + 32 * j < k) pis[lane + 32 * j] = pi[j];
                __syncwarp();
                double g[KJ];
#pragma unroll
                for (int j = 0; j < KJ; ++j) g[j] = 0.0;
                for (int b = 0; b < k; ++b) {
                    const double pb = pis[b];
                    const double* col = G + static_cast<size_t>(b) * k;
#pragma unroll
                    for (int j = 0; j < KJ; ++j)
                        if (lane + 32 * j < k) g[j] += col[lane + 32 * j] * pb;
                }
                __syncwarp();
                double nx[KJ];
#pragma unroll
                for (int j = 0; j < KJ; ++j) nx[j] = pi[j] - step * (g[j] - phi_tw[j]);
                warp_simplex<KJ>(nx, k);
                double moved = 0.0;
#pragma unroll
                for (int j = 0; j < KJ; ++j)
                    if (lane + 32 * j < k) moved += (nx[j] - pi[j]) * (nx[j] - pi[j]);
                moved = warp_sum(moved);
#pragma unroll
                for (int j = 0; j < KJ; ++j) pi[j] = nx[j];
                if (sqrt(moved) <= 1e-8) break;
            }
        }
        double ll = 0.0;
        long long fl = 0;
        for (long long q = q0; q < q1; ++q) {
            const double* row = Phi + static_cast<size_t>(word[q]) * k;
            double pw = 0.0;
#pragma unroll
            for (int j = 0; j < KJ; ++j)
                if (lane + 32 * j < k) pw += row[lane + 32 * j] * (k > 1 ? pi[j] : 1.0);
            pw = warp_sum(pw);
            if (pw < 1e-12) {
                pw = 1e-12;
                ++fl;
            }
            ll += count[q] * log(pw);
        }
        if (lane == 0) {
            per[d] = ll / static_cast<double>(tot);
            floored[d] = fl;
        }
    }
}

bool launch_lda_heldout(cudaStream_t st, int k, long long D, const long long* doc_ptr, const int* word, const int* count,
                        const double* Phi, const double* G, double step, double* per, long long* floored) {
    const size_t smem = sizeof(double) * (static_cast<size_t>(k) * k + 8ull * k);
    if (k > 128 || smem > 227 * 1024) return false;
    const unsigned grid = static_cast<unsigned>(std::min<long long>((D + 7) / 8, 148ll * 8));
#define HL_(KJ)                                                                                                    \
    {                                                                                                              \
        cudaFuncSetAttribute(k_heldout_docs<KJ>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)); \
        k_heldout_docs<KJ><<<grid, 256, smem, st>>>(k, D, doc_ptr, word, count, Phi, G, step, per, floored);     \
    }
    if (k <= 32) HL_(1) else if (k <= 64) HL_(2) else if (k <= 96) HL_(3) else HL_(4)
#undef HL_
    count_launch();
    return true;
}

}  // namespace skc
