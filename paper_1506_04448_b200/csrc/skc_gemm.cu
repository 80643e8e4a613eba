// FP64 block products of the LDA whitening and the fast-ALS normal equations, on sm_100a.
//
// The whitening (lda.cpp:88-143, randomized subspace iteration in skc_abi_lda.cu) and the
// ALS update (decompose.cpp:117-208) need four product shapes, all C = op(A) op(B) with
// alpha 1 and beta 0: the Gram of a tall block (p x p from V x p, K = V = 5e4 at config 4),
// a small matrix applied to a wide block (p x V from p x p and p x V), the dense V x V
// moment applied to a block, and the k x k Grams / n x k update of ALS. One kernel with
// element strides covers them: 64 x 64 output tiles, 16-deep k slabs staged in shared
// memory k-major (each thread's 4 x 4 outputs read as two 16-byte vectors per operand per
// k step), the next slab's loads in registers while the current one is multiplied. Short,
// deep products (the Grams: 4 tiles, K = 5e4) are split along K into a fixed number of
// slices whose partial tiles are summed in slice order by a second kernel, so results are
// deterministic run to run.
#include <cuda_runtime.h>

#include <algorithm>

#include "skc_internal.hpp"

namespace skc {

namespace {
constexpr int BM = 64, BN = 64, BK = 16, NT = 256;

// A(i, l) = A[i * ai + l * ak], B(l, j) = B[l * bk + j * bj]; slice z covers l in
// [z * kc, min(K, (z + 1) * kc)). Output tile to C(i, j) = C[i * ci + j * cj] (one slice) or
// to the slice's partial plane W[z][i][j] (M x N row-major).
__global__ void __launch_bounds__(NT) k_dgemm(const double* __restrict__ A, long long ai, long long ak,
                                              const double* __restrict__ B, long long bk, long long bj, int M, int N,
                                              int K, int kc, double* __restrict__ C, long long ci, long long cj) {
    __shared__ __align__(16) double As[BK][BM];
    __shared__ __align__(16) double Bs[BK][BN];
    const int t = threadIdx.x, tx = t & 15, ty = t >> 4;
    const int i0 = blockIdx.y * BM, j0 = blockIdx.x * BN;
    const int l0 = blockIdx.z * kc, l1 = min(K, l0 + kc);
    // staging map: the unit-stride index runs across consecutive threads (coalesced)
    const bool a_irow = ai == 1, b_jrow = bj == 1;
    double ra[4], rb[4];
    auto load = [&](int lb) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int e = t + NT * q;
            const int ii = a_irow ? (e & (BM - 1)) : (e >> 4), la = a_irow ? (e >> 6) : (e & (BK - 1));
            const int i = i0 + ii, l = lb + la;
            ra[q] = (i < M && l < l1) ? __ldg(A + i * ai + l * ak) : 0.0;
            const int jj = b_jrow ? (e & (BN - 1)) : (e >> 4), lbb = b_jrow ? (e >> 6) : (e & (BK - 1));
            const int j = j0 + jj, l2 = lb + lbb;
            rb[q] = (j < N && l2 < l1) ? __ldg(B + l2 * bk + j * bj) : 0.0;
        }
    };
    auto store = [&]() {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int e = t + NT * q;
            const int ii = a_irow ? (e & (BM - 1)) : (e >> 4), la = a_irow ? (e >> 6) : (e & (BK - 1));
            As[la][ii] = ra[q];
            const int jj = b_jrow ? (e & (BN - 1)) : (e >> 4), lbb = b_jrow ? (e >> 6) : (e & (BK - 1));
            Bs[lbb][jj] = rb[q];
        }
    };
    double acc[4][4] = {};
    if (l0 < l1) load(l0);
    for (int lb = l0; lb < l1; lb += BK) {
        __syncthreads();
        store();
        __syncthreads();
        if (lb + BK < l1) load(lb + BK);
#pragma unroll
        for (int l = 0; l < BK; ++l) {
            const double2 a01 = *reinterpret_cast<const double2*>(&As[l][ty * 4]);
            const double2 a23 = *reinterpret_cast<const double2*>(&As[l][ty * 4 + 2]);
            const double2 b01 = *reinterpret_cast<const double2*>(&Bs[l][tx * 4]);
            const double2 b23 = *reinterpret_cast<const double2*>(&Bs[l][tx * 4 + 2]);
            const double a[4] = {a01.x, a01.y, a23.x, a23.y}, b[4] = {b01.x, b01.y, b23.x, b23.y};
#pragma unroll
            for (int r = 0; r < 4; ++r)
#pragma unroll
                for (int c = 0; c < 4; ++c) acc[r][c] = fma(a[r], b[c], acc[r][c]);
        }
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        const int i = i0 + ty * 4 + r;
        if (i >= M) continue;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const int j = j0 + tx * 4 + c;
            if (j >= N) continue;
            if (gridDim.z == 1) C[i * ci + j * cj] = acc[r][c];
            else C[(static_cast<long long>(blockIdx.z) * M + i) * N + j] = acc[r][c];
        }
    }
}

// C(i, j) = sum over slices z = 0, 1, ... of W[z][i][j], in slice order
__global__ void k_dgemm_reduce(const double* __restrict__ W, int slices, int M, int N, double* __restrict__ C,
                               long long ci, long long cj) {
    const long long e = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= static_cast<long long>(M) * N) return;
    double s = 0.0;
    for (int z = 0; z < slices; ++z) s += W[static_cast<long long>(z) * M * N + e];
    const int i = static_cast<int>(e / N), j = static_cast<int>(e - static_cast<long long>(i) * N);
    C[i * ci + j * cj] = s;
}
}  // namespace

int dgemm_slices(int M, int N, int K, int sms) {
    const long long tiles = static_cast<long long>((M + BM - 1) / BM) * ((N + BN - 1) / BN);
    if (tiles >= sms) return 1;
    const long long want = (2LL * sms + tiles - 1) / tiles;
    // (slices of at least 64: the ALS Grams, k x k from n ~ 1000 rows, would otherwise be one
    // CTA walking 60 dependent slabs)
    return static_cast<int>(std::max(1LL, std::min<long long>(want, K / 64)));
}

void launch_dgemm(cudaStream_t st, int sms, int M, int N, int K, const double* A, long long ai, long long ak,
                  const double* B, long long bk, long long bj, double* C, long long ci, long long cj, double* ws) {
    if (M <= 0 || N <= 0) return;
    const int z = (K > 0) ? dgemm_slices(M, N, K, sms) : 1;
    const int kc = z > 1 ? ((K + z - 1) / z + BK - 1) / BK * BK : std::max(K, 1);
    const int zz = z > 1 ? (K + kc - 1) / kc : 1;
    const dim3 grid((N + BN - 1) / BN, (M + BM - 1) / BM, zz);
    if (zz == 1) {
        k_dgemm<<<grid, NT, 0, st>>>(A, ai, ak, B, bk, bj, M, N, K, kc, C, ci, cj);
        count_launch();
        return;
    }
    k_dgemm<<<grid, NT, 0, st>>>(A, ai, ak, B, bk, bj, M, N, K, kc, ws, 0, 0);
    count_launch();
    const long long mn = static_cast<long long>(M) * N;
    k_dgemm_reduce<<<static_cast<unsigned>((mn + 255) / 256), 256, 0, st>>>(ws, zz, M, N, C, ci, cj);
    count_launch();
}

}  // namespace skc
