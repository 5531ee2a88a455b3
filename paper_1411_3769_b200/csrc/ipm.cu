// ipm.cu -- polya_ipm_step: one predictor-corrector iteration of Algorithm 2
// with the readings R3-R6 of DESIGN.md, on one GPU.  Every iterate is a block stack
// double[nblocks][n][n] (Theorem 3: the iteration never leaves S_{L,M,n}).
//
//   W   = Z^-1 (blockwise Cholesky inverse)                 kernel k_block_inv
//   Rd  = -B^T(y) + Z + C                                   (Eq. G; polya_apply + k_axpby)
//   O1  = B(W Rd X) - 1                                     (Processors step 1, Eq. T1)
//   G   = SCM (polya_schur, POLYA_G_FULL)                   (Eq. T2)
//   potrf(G); dy^ = G^-1 O1                                 (Root step 1, Eq. SAE1; cuSOLVER)
//     -- or, when the K x K matrix does not fit (config 5: 186 GB), a right-looking block Cholesky
//        over the PAIR_TILES layout of polya_schur (cuSOLVER potrf on diagonal tiles, cuBLAS
//        trsm / syrk / gemm on the rest) and blocked triangular solves: the root's factorisation
//        (Case 2) on one GPU with half the memory
//   dZ^ = -Rd + B^T(dy^);  dX^ = sym(-X + W (Rd - B^T(dy^)) X)          (R3)
//   O2  = mu B(W) - B(W dZ^ dX^);  dy- = G^-1 O2            (Processors/Root step 2, Eq. SAE2)
//   dZ- = B^T(dy-);  dX- = sym(mu W - W dZ^ dX^ - W dZ- X)  (Processors step 3)
//   t_p, t_d = min(1, 0.98 t_max), t_max by per-block bisection on positive definiteness (R5)
//   X += t_p dX, Z += t_d dZ, y += t_d dy                   (Eqs. 33-35, R6)
//   mu = tr(ZX) / (3 (L+M) n) (R4), phi = tr(CX), psi = sum y, gap = |phi - psi|   (Step 4)
#include <cublas_v2.h>
#include <cusolverDn.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "polya_internal.h"

namespace polya {
namespace {

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// C_b = alpha op(A_b) op(B_b) + beta C_b for every block b of n x n stacks (any n; guarded loads).
// CTA = 32x32 tile of one block, 4 warps of 2x2 DMMA m8n8 tiles, K staged 8 at a time.
__global__ void __launch_bounds__(128) k_bgemm(int n, const double* __restrict__ A, int ta,
                                               const double* __restrict__ B, int tb, double* __restrict__ C,
                                               double alpha, double beta, int tiles) {
  __shared__ double As[8][40];
  __shared__ double Bs[8][40];
  const int64_t nn = (int64_t)n * n, b = blockIdx.y;
  const double* Ab = A + b * nn;
  const double* Bb = B + b * nn;
  double* Cb = C + b * nn;
  const int ti = blockIdx.x / tiles, tj = blockIdx.x - ti * tiles, i0 = ti * 32, j0 = tj * 32;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, t = lane & 3;
  const int wr = (warp >> 1) * 16, wc = (warp & 1) * 16;
  double acc[2][2][2] = {};
  for (int k0 = 0; k0 < n; k0 += 8) {
    for (int e = tid; e < 256; e += 128) {
      const int r = e >> 3, k = e & 7;  // A tile: rows i0+r, k0+k
      const int gi = i0 + r, gk = k0 + k;
      As[k][r] = (gi < n && gk < n) ? (ta ? Ab[(int64_t)gk * n + gi] : Ab[(int64_t)gi * n + gk]) : 0.0;
      const int gj = j0 + r;             // B tile: k0+k, cols j0+r
      Bs[k][r] = (gj < n && gk < n) ? (tb ? Bb[(int64_t)gj * n + gk] : Bb[(int64_t)gk * n + gj]) : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {
      double a[2], bb[2];
#pragma unroll
      for (int mi = 0; mi < 2; ++mi) a[mi] = As[ks * 4 + t][wr + mi * 8 + g];
#pragma unroll
      for (int nj = 0; nj < 2; ++nj) bb[nj] = Bs[ks * 4 + t][wc + nj * 8 + g];
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int nj = 0; nj < 2; ++nj) dmma(acc[mi][nj][0], acc[mi][nj][1], a[mi], bb[nj]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int nj = 0; nj < 2; ++nj)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int i = i0 + wr + mi * 8 + g, j = j0 + wc + nj * 8 + 2 * t + e;
        if (i < n && j < n) {
          const int64_t o = (int64_t)i * n + j;
          Cb[o] = alpha * acc[mi][nj][e] + (beta != 0.0 ? beta * Cb[o] : 0.0);
        }
      }
}

// out = a X + b Y (+ c * C_b on the P-blocks' diagonals when cdiag != nullptr), elementwise
__global__ void k_axpby(int64_t total, int n, int nbas, int64_t Lp, double a, const double* __restrict__ X, double b,
                        const double* __restrict__ Y, double* __restrict__ out, const double* __restrict__ cdiag,
                        double cs, const double* __restrict__ cL) {
  const int64_t nn = (int64_t)n * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    double v = a * X[e] + (Y ? b * Y[e] : 0.0);
    if (cdiag) {   // C: c_j I on the P-blocks, the dense C_L (generalised form's R) on the Lyapunov blocks
      const int64_t blk = e / nn, r = e - blk * nn;
      if (blk < Lp && (r / n) == (r % n)) v += cs * ((r / n) < nbas ? cdiag[blk] : -1.0);   // -I: padding (R19)
      if (blk >= Lp && cL) v += cs * cL[e - Lp * nn];
    }
    out[e] = v;
  }
}

// out_b = (M_b + M_b^T) / 2
__global__ void k_sym(int n, const double* __restrict__ M, double* __restrict__ out) {
  const int64_t nn = (int64_t)n * n, b = blockIdx.x;
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    const int i = e / n, j = e - i * n;
    if (i <= j) {
      const double v = 0.5 * (M[b * nn + (int64_t)i * n + j] + M[b * nn + (int64_t)j * n + i]);
      out[b * nn + (int64_t)i * n + j] = v;
      out[b * nn + (int64_t)j * n + i] = v;
    }
  }
}

// In-shared-memory Cholesky of the n x n matrix S (row-major, lower factor in place).
// Returns false (uniformly) if a pivot is not positive.
__device__ bool smem_chol(double* S, int n) {
  __shared__ int s_ok;
  if (threadIdx.x == 0) s_ok = 1;
  __syncthreads();
  for (int k = 0; k < n; ++k) {
    if (threadIdx.x == 0) {
      const double d = S[k * n + k];
      if (!(d > 0.0)) s_ok = 0;
      S[k * n + k] = d > 0.0 ? sqrt(d) : 1.0;
    }
    __syncthreads();
    if (!s_ok) return false;
    const double dk = S[k * n + k];
    for (int i = k + 1 + threadIdx.x; i < n; i += blockDim.x) S[i * n + k] /= dk;
    __syncthreads();
    for (int e = threadIdx.x; e < (n - k - 1) * (n - k - 1); e += blockDim.x) {
      const int i = k + 1 + e / (n - k - 1), j = k + 1 + e % (n - k - 1);
      if (j <= i) S[i * n + j] -= S[i * n + k] * S[j * n + k];
    }
    __syncthreads();
  }
  return true;
}

// W_b = Z_b^{-1} via Cholesky Z = L L^T, X = L^{-1} in place, then W = X^T X (exactly symmetric).
// One CTA per block, every phase right-looking with one barrier per column: the Cholesky (column k's
// rank-1 update of the trailing triangle with the column scaled on the fly; the stored column is scaled
// during the next column's update, which does not touch it), the inverse (L X = I by rows: the update
// of step k also finishes row k+1 of X), and X^T X in 2x2 register blocks.  Rows in shared memory with
// an odd stride (n | 1 doubles), so the column reads of a half-warp hit distinct banks.
// Shared memory: n (n | 1) + 3n doubles (n <= 168).
// linv != 0: W_b = L^{-1} instead (lower triangle, zeros above; a NaN in W_b[0] if Z_b is not positive
// definite), the congruence factor of the step length (step_len).
__global__ void __launch_bounds__(512, 2) k_block_inv(int n, const double* __restrict__ Z, double* __restrict__ W,
                                                   int* __restrict__ fail, int linv = 0) {
  extern __shared__ double sm[];
  const int ld = n | 1, tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  double* S = sm;                  // n x ld: Z, then L (lower), then X = L^{-1} (lower)
  double* dinv = S + n * ld;       // 1 / L_kk
  double* colb = dinv + n;         // two buffers of a column of L (the inverse's right-looking update)
  const int64_t nn = (int64_t)n * n, b = blockIdx.x;
  for (int i = warp; i < n; i += nw)
    for (int j = lane; j < n; j += 32) S[i * ld + j] = Z[b * nn + (int64_t)i * n + j];
  __syncthreads();
  // ---- Cholesky, lower: L_kk = sqrt(p_k), L_ik = S_ik / L_kk, S_ij -= L_ik L_jk (k < j <= i)
  double rs_prev = 0.0, sq_prev = 0.0;
  for (int k = 0; k < n; ++k) {
    const double piv = S[k * ld + k];
    if (!(piv > 0.0)) {   // every thread read the same pivot: a uniform exit
      if (tid == 0) {
        if (fail) atomicExch(fail, 1);
        if (linv) W[b * nn] = __longlong_as_double(0x7ff8000000000000LL);
      }
      return;
    }
    const double sq = sqrt(piv), rs = 1.0 / sq;
    for (int i = k + 1 + warp; i < n; i += nw) {
      const double lik = S[i * ld + k] * rs;
      for (int j = k + 1 + lane; j <= i; j += 32) S[i * ld + j] -= lik * (S[j * ld + k] * rs);
    }
    if (k > 0) {   // column k-1 (read only by step k-1's update) takes its final scaling
      for (int i = k + tid; i < n; i += nt) S[i * ld + k - 1] *= rs_prev;
      if (tid == 0) { S[(k - 1) * ld + k - 1] = sq_prev; dinv[k - 1] = rs_prev; }
    }
    rs_prev = rs;
    sq_prev = sq;
    __syncthreads();
  }
  if (tid == 0) { S[(n - 1) * ld + n - 1] = sq_prev; dinv[n - 1] = rs_prev; }
  // ---- X = L^{-1}, lower, by rows: X_kj = B_kj / L_kk with B = I - sum_{m<k} L_km X_mj accumulated
  // right-looking in the storage of L's consumed columns (position (r, j), j <= k < r, holds B_rj)
  if (tid == 0) S[0] = dinv[0];
  for (int r = 1 + tid; r < n; r += nt) colb[r] = S[r * ld];       // column 0 of L
  __syncthreads();
  for (int k = 0; k + 1 < n; ++k) {
    const double* cur = colb + (k & 1) * n;
    double* nxt = colb + ((k + 1) & 1) * n;
    const int w = k + 1, cnt = (n - k - 1) * w;
    const double dn = dinv[k + 1];
    for (int e = tid; e < cnt; e += nt) {
      const int q = e / w, j = e - q * w, r = k + 1 + q;
      double v = (j == k ? 0.0 : S[r * ld + j]) - cur[r] * S[k * ld + j];
      if (r == k + 1) v *= dn;   // row k+1 of X is final after this update
      S[r * ld + j] = v;
    }
    for (int r = k + 2 + tid; r < n; r += nt) nxt[r] = S[r * ld + k + 1];   // column k+1 of L (untouched here)
    if (tid == 0) S[(k + 1) * ld + k + 1] = dn;
    __syncthreads();
  }
  if (linv) {
    for (int i = warp; i < n; i += nw)
      for (int j = lane; j < n; j += 32) W[b * nn + (int64_t)i * n + j] = j <= i ? S[i * ld + j] : 0.0;
    return;
  }
  for (int i = warp; i < n; i += nw)   // the strict upper triangle of X is zero
    for (int j = i + 1 + lane; j < n; j += 32) S[i * ld + j] = 0.0;
  __syncthreads();
  // ---- W = X^T X: W_ij = sum_{m >= max(i,j)} X_mi X_mj, 2x2 blocks (I <= J) of (i, j) = (2I.., 2J..)
  const int h = (n + 1) >> 1, nblk = h * (h + 1) / 2;
  for (int e = tid; e < nblk; e += nt) {
    int J = (int)((sqrt(8.0 * e + 1.0) - 1.0) * 0.5);   // e = J (J + 1) / 2 + I, I <= J
    while (J * (J + 1) / 2 > e) --J;
    while ((J + 1) * (J + 2) / 2 <= e) ++J;
    const int I = e - J * (J + 1) / 2;
    const int i0 = 2 * I, i1 = i0 + 1, j0 = 2 * J, j1 = j0 + 1;
    const bool vi = i1 < n, vj = j1 < n;
    double w00 = 0.0, w01 = 0.0, w10 = 0.0, w11 = 0.0;
    for (int m = j0; m < n; ++m) {
      const double* row = S + m * ld;
      const double a0 = row[i0], a1 = vi ? row[i1] : 0.0, c0 = row[j0], c1 = vj ? row[j1] : 0.0;
      w00 = fma(a0, c0, w00);
      w01 = fma(a0, c1, w01);
      w10 = fma(a1, c0, w10);
      w11 = fma(a1, c1, w11);
    }
    double* Wb = W + b * nn;
    Wb[(int64_t)i0 * n + j0] = w00;
    Wb[(int64_t)j0 * n + i0] = w00;
    if (vj) { Wb[(int64_t)i0 * n + j1] = w01; Wb[(int64_t)j1 * n + i0] = w01; }
    if (vi) { Wb[(int64_t)i1 * n + j0] = w10; Wb[(int64_t)j0 * n + i1] = w10; }
    if (vi && vj) { Wb[(int64_t)i1 * n + j1] = w11; Wb[(int64_t)j1 * n + i1] = w11; }
  }
}

size_t block_inv_smem(int64_t n) { return ((size_t)n * (size_t)(n | 1) + 3 * (size_t)n) * sizeof(double); }

// Reading R5 as written: t_b = min(tcap, 1 / max(0, -lambda_min(M_b))), M_b = L_b^{-1} dS_b L_b^{-T}
// (S_b = L_b L_b^T; M_b formed by k_block_inv(linv) + two k_bgemm).  One CTA (512 threads) per block:
// the symmetric part of M_b, in full storage in shared memory (n (n|1) + 3n doubles, n <= 168), is
// reduced to tridiagonal form by Householder reflections (A <- H A H, H = I - tau v v^T; LAPACK
// dsytd2's algorithm), then lambda_min by multisection on the Sturm count of the tridiagonal (512
// trial points per round, one per thread).  Non-finite M_b (S_b not positive definite, e.g. a singular X on the
// boundary of the cone): t_b = -1, for which step_len runs the bisection kernel k_block_tmax.
// Number of eigenvalues of the symmetric tridiagonal T below lam (Sturm sequence of T - lam I); the
// diagonal d_i = T[i * st], the off-diagonal e_i = T[i * st + 1] (the tridiagonal kept in place in the
// reduced matrix: st = ld + 1).
__device__ __forceinline__ int sturm_count(int n, const double* T, int st, double lam) {
  int cnt = 0;
  double q = T[0] - lam;
  for (int i = 0;; ++i) {
    if (q == 0.0) q = -1e-300;
    cnt += q < 0.0;
    if (i + 1 == n) break;
    const double ei = T[i * st + 1];
    q = (T[(i + 1) * st] - lam) - ei * ei / q;
  }
  return cnt;
}
// Shared-memory row stride of k_block_lmin: odd (conflict-free column reads) when it fits.
__host__ __device__ inline int lmin_ld(int n) {
  return ((int64_t)n * (n | 1) + 3 * n) * 8 + 512 <= 232448 ? (n | 1) : n;
}
size_t block_lmin_smem(int64_t n) { return ((size_t)n * lmin_ld((int)n) + 3 * (size_t)n) * sizeof(double); }

__global__ void __launch_bounds__(512, 2) k_block_lmin(int n, const double* __restrict__ M, double tcap,
                                                    double* __restrict__ tout) {
  extern __shared__ double sm[];
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  const int ld = lmin_ld(n);
  double* A = sm;            // n x ld, full symmetric storage of sym(M_b)
  double* p = A + n * ld;    // tau A v on the trailing block
  double* vc = p + n;        // two buffers of the Householder vector
  // the tridiagonal stays in place: d_k = A_kk (final after step k-1), e_k in A_{k,k+1} (the upper
  // triangle of row k, dead once step k starts)
  __shared__ double red[32];
  __shared__ int s_j;
  const int64_t b = blockIdx.x, nn = (int64_t)n * n;
  const double* Mb = M + b * nn;
  int bad = 0;
  for (int i = warp; i < n; i += nw)
    for (int j = lane; j < n; j += 32) {
      const double x = 0.5 * (Mb[(int64_t)i * n + j] + Mb[(int64_t)j * n + i]);
      bad |= !isfinite(x);
      A[i * ld + j] = x;
    }
  if (__syncthreads_or(bad)) {
    if (tid == 0) tout[b] = -1.0;   // S_b not positive definite: step_len falls back to k_block_tmax
    return;
  }
  // Householder (LAPACK dsytd2's reflections, A <- H A H, H = I - tau v v^T), two barriers per column.
  // v is column k below the diagonal, in vc[k & 1] (written by the previous column's update, which
  // finishes column k), with v_{k+1} = x_0 - e_k substituted where it is read.  The column norm and p^T v
  // are reduced redundantly by every warp (shuffles).
  for (int i = 1 + tid; i < n; i += nt) vc[i] = A[i * ld];
  __syncthreads();
  for (int k = 0; k + 2 < n; ++k) {
    const int k1 = k + 1;
    double* v = vc + (k & 1) * n;
    double* vn = vc + ((k + 1) & 1) * n;
    double xs = 0.0;
    for (int i = k1 + lane; i < n; i += 32) xs = fma(v[i], v[i], xs);
    for (int o = 16; o > 0; o >>= 1) xs += __shfl_xor_sync(0xffffffffu, xs, o);
    const double a2 = xs, x0 = v[k1];
    const double alpha = sqrt(a2), ek = x0 >= 0.0 ? -alpha : alpha;
    if (tid == 0) A[k * ld + k1] = ek;
    if (a2 == 0.0) {   // already reduced (uniform): column k+1 for the next step
      for (int i = k1 + 1 + tid; i < n; i += nt) vn[i] = A[i * ld + k1];
      __syncthreads();
      continue;
    }
    const double v0 = x0 - ek, tau = 2.0 / (a2 - x0 * x0 + v0 * v0);
    // p_i = tau sum_j A_ij v_j (rows i > k, two threads per row: half-warps of 16 rows)
    for (int base = k1 + warp * 16; base < n; base += nw * 16) {
      const int i = base + (lane & 15), half = lane >> 4;
      double a0 = 0.0, a1 = 0.0;
      if (i < n) {
        const double* Ai = A + i * ld;
        if (half == 0) a0 = Ai[k1] * v0;
        int j = k1 + 1 + half;
        for (; j + 2 < n; j += 4) {
          a0 = fma(Ai[j], v[j], a0);
          a1 = fma(Ai[j + 2], v[j + 2], a1);
        }
        if (j < n) a0 = fma(Ai[j], v[j], a0);
      }
      double acc = a0 + a1;
      acc += __shfl_xor_sync(0xffffffffu, acc, 16);
      if (i < n && half == 0) p[i] = tau * acc;
    }
    __syncthreads();
    double pv = (lane == 0) ? p[k1] * v0 : 0.0;
    for (int i = k1 + 1 + lane; i < n; i += 32) pv = fma(p[i], v[i], pv);
    for (int o = 16; o > 0; o >>= 1) pv += __shfl_xor_sync(0xffffffffu, pv, o);
    const double Kc = 0.5 * tau * pv;
    // A <- A - v w^T - w v^T on the trailing block (both triangles, bitwise symmetric), w = p - K v;
    // column k+1 of the result is the next step's v
    for (int i = k1 + warp; i < n; i += nw) {
      const double vi = i == k1 ? v0 : v[i], wi = p[i] - Kc * vi;
      double* Ai = A + i * ld;
      for (int j = k1 + lane; j < n; j += 32) {
        const double vj = j == k1 ? v0 : v[j], wj = p[j] - Kc * vj;
        const double r = Ai[j] - __dadd_rn(__dmul_rn(vi, wj), __dmul_rn(wi, vj));
        Ai[j] = r;
        if (j == k1 && i > k1) vn[i] = r;
      }
    }
    __syncthreads();
  }
  __syncthreads();   // e_{n-2} = A_{n-2,n-1} (the symmetric copy of the last reflection's result)
  // lambda_min >= 0: no bound on t (tcap); else multisection on [Gershgorin lower bound, 0]
  const int st = ld + 1;
  if (sturm_count(n, A, st, 0.0) == 0) {
    if (tid == 0) tout[b] = tcap;
    return;
  }
  double lo = 0.0;
  {
    double g = 1e300;
    for (int i = tid; i < n; i += nt)
      g = fmin(g, A[i * st] - (i > 0 ? fabs(A[(i - 1) * st + 1]) : 0.0) - (i + 1 < n ? fabs(A[i * st + 1]) : 0.0));
    for (int o = 16; o > 0; o >>= 1) g = fmin(g, __shfl_xor_sync(0xffffffffu, g, o));
    if (lane == 0) red[warp] = g;
    __syncthreads();
    for (int q = 0; q < nw; ++q) lo = fmin(lo, red[q]);
    lo -= 1e-12 * fabs(lo) + 1e-300;
  }
  double hi = 0.0;
  for (int round = 0; round < 12 && hi - lo > 4e-16 * fmax(fabs(lo), fabs(hi)); ++round) {
    const double step = (hi - lo) / (double)(nt + 1);
    const double lam = lo + step * (tid + 1);
    const int below = sturm_count(n, A, st, lam) == 0;   // lam <= lambda_min
    if (tid == 0) s_j = -1;
    __syncthreads();
    if (below) atomicMax(&s_j, tid);
    __syncthreads();
    const int j = s_j;
    const double nlo = lo + step * (j + 1), nhi = j + 1 < nt ? lo + step * (j + 2) : hi;
    lo = nlo;
    hi = nhi;
    __syncthreads();
  }
  if (tid == 0) tout[b] = fmin(tcap, -1.0 / (0.5 * (lo + hi)));
}

// Fallback of step_len for a block with S_b only semidefinite (no L_b^{-1}): t_b = sup{t in [0, tcap] :
// S_b + t dS_b positive definite} by bisection on the Cholesky test (60 halvings); blocks with
// tout[b] >= 0 already are skipped.
__global__ void k_block_tmax(int n, const double* __restrict__ S, const double* __restrict__ dS, double tcap,
                             double* __restrict__ tout) {
  extern __shared__ double sm[];
  const int64_t nn = (int64_t)n * n, b = blockIdx.x;
  if (tout[b] >= 0.0) return;
  auto pd = [&](double tt) -> bool {
    for (int e = threadIdx.x; e < n * n; e += blockDim.x) sm[e] = S[b * nn + e] + tt * dS[b * nn + e];
    __syncthreads();
    const bool ok = smem_chol(sm, n);
    __syncthreads();
    return ok;
  };
  double lo = 0.0, hi = tcap;
  if (pd(hi)) {
    lo = hi;
  } else {
    for (int it = 0; it < 60; ++it) {
      const double mid = 0.5 * (lo + hi);
      if (pd(mid)) lo = mid; else hi = mid;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) tout[b] = lo;
}

// partial sums: out[0] = sum_b tr(Z_b X_b) = sum Z.*X^T, out[1] = sum_{j<L} c_j tr(X_j), out[2] = sum y
__global__ void k_scalars(int64_t total, int n, int nbas, int64_t Lp, const double* __restrict__ Z, const double* __restrict__ X,
                          const double* __restrict__ c, const double* __restrict__ y, int64_t K,
                          double* __restrict__ part, const double* __restrict__ cL) {
  __shared__ double red[3][256];
  const int64_t nn = (int64_t)n * n;
  double s0 = 0, s1 = 0, s2 = 0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t blk = e / nn, r = e - blk * nn;
    const int i = (int)(r / n), j = (int)(r % n);
    s0 += Z[e] * X[blk * nn + (int64_t)j * n + i];
    if (blk < Lp && i == j) s1 += (i < nbas ? c[blk] : -1.0) * X[e];
    if (blk >= Lp && cL) s1 += cL[e - Lp * nn] * X[blk * nn + (int64_t)j * n + i];   // tr(C_L X)
  }
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < K; e += (int64_t)gridDim.x * blockDim.x) s2 += y[e];
  red[0][threadIdx.x] = s0; red[1][threadIdx.x] = s1; red[2][threadIdx.x] = s2;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w)
      for (int q = 0; q < 3; ++q) red[q][threadIdx.x] += red[q][threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0)
    for (int q = 0; q < 3; ++q) part[blockIdx.x * 3 + q] = red[q][0];
}

__global__ void k_vec_axpby(int64_t K, double a, const double* __restrict__ x, double b, const double* __restrict__ y,
                            double* __restrict__ out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < K; e += (int64_t)gridDim.x * blockDim.x)
    out[e] = a * x[e] + (y ? b * y[e] : 0.0);
}

__global__ void k_vec_shift(int64_t K, double cst, double* __restrict__ x) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < K; e += (int64_t)gridDim.x * blockDim.x)
    x[e] += cst;
}

// part[blk] = partial sum of (v_e - 1)^2 (primal residual ||B(X) - a||^2, a = 1)
__global__ void k_resid(int64_t K, const double* __restrict__ v, double* __restrict__ part) {
  __shared__ double red[256];
  double s = 0.0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < K; e += (int64_t)gridDim.x * blockDim.x) {
    const double d = v[e] - 1.0;
    s += d * d;
  }
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}

// X_b = Z_b = I (Algorithm 2's initial point)
__global__ void k_identity(int64_t total, int n, double* __restrict__ X, double* __restrict__ Z) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e % ((int64_t)n * n);
    const double v = (r / n == r % n) ? 1.0 : 0.0;
    X[e] = v;
    Z[e] = v;
  }
}

// Verdict grid check (O8, Theorem 1): at the point alpha = pts[blockIdx.x] of the simplex,
//   P(alpha) = sum_h alpha^h V_h(y)   (reading R7; V_h in the arena after k_vmap)
//   A(alpha) = sum_lambda alpha^lambda A_lambda
// and the test P(alpha) > 0, -(A^T P + P A)(alpha) > 0 by Cholesky.  P(alpha), A(alpha) and the
// Lyapunov matrix live in a per-point global scratch (3 n^2); each Cholesky test runs on a copy in
// shared memory (n^2 doubles: n <= 168, the IPM's limit).
__device__ bool chol_copy(double* C, const double* src, int n, int ld) {
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) C[e] = src[(e / n) * ld + (e % n)];
  __syncthreads();
  const bool ok = smem_chol(C, n);
  __syncthreads();
  return ok;
}

__global__ void k_grid(int n, int l, int L0, int nA, const int32_t* __restrict__ Wp, const int32_t* __restrict__ Wa,
                       const double* __restrict__ arena, int64_t ms, int np, int64_t id_Vy,
                       const double* __restrict__ A, const double* __restrict__ pts, double* __restrict__ scratch,
                       int* __restrict__ nfail) {
  extern __shared__ double sm[];
  double* C = sm;                  // n^2: Cholesky work matrix
  double* mono = sm + n * n;       // [L0 + nA]
  const int64_t nn = (int64_t)n * n;
  double* P = scratch + (int64_t)blockIdx.x * 3 * nn;
  double* Aa = P + nn;
  double* M = Aa + nn;
  const double* al = pts + (int64_t)blockIdx.x * l;
  for (int q = threadIdx.x; q < L0 + nA; q += blockDim.x) {
    const int32_t* e = q < L0 ? Wp + (int64_t)q * l : Wa + (int64_t)(q - L0) * l;
    double m = 1.0;
    for (int i = 0; i < l; ++i)
      for (int k = 0; k < e[i]; ++k) m *= al[i];
    mono[q] = m;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    const int i = e / n, j = e - i * n;
    double p = 0.0, a = 0.0;
    for (int h = 0; h < L0; ++h) p += mono[h] * arena[(id_Vy + h) * ms + (int64_t)i * np + j];
    for (int q = 0; q < nA; ++q) a += mono[L0 + q] * A[(int64_t)q * n * n + e];
    P[e] = p;
    Aa[e] = a;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    const int i = e / n, j = e - i * n;
    double v = 0.0;
    for (int k = 0; k < n; ++k) v += Aa[k * n + i] * P[k * n + j] + P[i * n + k] * Aa[k * n + j];
    M[e] = -v;
  }
  __syncthreads();
  const bool lyap = chol_copy(C, M, n, n);
  const bool pos = chol_copy(C, P, n, n);
  if (threadIdx.x == 0 && !(lyap && pos)) atomicAdd(nfail, 1);
}

// The same check for the generalised form (reading R18): -sum_i (At_i P Bt_i + transpose)(alpha) - R > 0
// (n = block order; the positivity test on P's nbas x nbas corner, R19).  Global scratch per point:
// P(alpha), the accumulator S = sum_i At_i P Bt_i, At_i(alpha), Bt_i(alpha), P Bt_i(alpha).
__global__ void k_grid_gen(int n, int nbas, int l, int L0, int nterms, int ncoef, int roff, const int32_t* __restrict__ Wp,
                           const int32_t* __restrict__ cexp, const int32_t* __restrict__ aoff,
                           const int32_t* __restrict__ boff, const double* __restrict__ coef,
                           const double* __restrict__ arena, int64_t ms, int np, int64_t id_Vy,
                           const double* __restrict__ pts, double* __restrict__ scratch, int* __restrict__ nfail) {
  extern __shared__ double sm[];
  double* C = sm;                  // n^2: Cholesky work matrix
  double* mono = sm + n * n;       // [L0 + ncoef]
  const int64_t nn = (int64_t)n * n;
  double* P = scratch + (int64_t)blockIdx.x * 5 * nn;
  double* S = P + nn;
  double* Ae = S + nn;
  double* Be = Ae + nn;
  double* PB = Be + nn;
  const double* al = pts + (int64_t)blockIdx.x * l;
  for (int q = threadIdx.x; q < L0 + ncoef; q += blockDim.x) {
    const int32_t* e = q < L0 ? Wp + (int64_t)q * l : cexp + (int64_t)(q - L0) * l;
    double m = 1.0;
    for (int i = 0; i < l; ++i)
      for (int k = 0; k < e[i]; ++k) m *= al[i];
    mono[q] = m;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    const int i = e / n, j = e - i * n;
    double p = 0.0;
    for (int h = 0; h < L0; ++h) p += mono[h] * arena[(id_Vy + h) * ms + (int64_t)i * np + j];
    P[e] = p;
    double r = 0.0;   // the constant term R(alpha), coefficients [roff, ncoef)
    for (int q = roff; q < ncoef; ++q) r += mono[L0 + q] * coef[q * nn + e];
    S[e] = 0.5 * r;
  }
  __syncthreads();
  for (int t = 0; t < nterms; ++t) {
    const int a0 = aoff[t], a1 = boff[t], b0 = boff[t], b1 = t + 1 < nterms ? aoff[t + 1] : roff;
    for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
      double a = 0.0, b = 0.0;
      for (int q = a0; q < a1; ++q) a += mono[L0 + q] * coef[q * nn + e];
      for (int q = b0; q < b1; ++q) b += mono[L0 + q] * coef[q * nn + e];
      Ae[e] = a;
      Be[e] = b;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
      const int i = e / n, j = e - i * n;
      double v = 0.0;
      for (int k = 0; k < n; ++k) v += P[i * n + k] * Be[k * n + j];
      PB[e] = v;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
      const int i = e / n, j = e - i * n;
      double v = 0.0;
      for (int k = 0; k < n; ++k) v += Ae[i * n + k] * PB[k * n + j];
      S[e] += v;
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    const int i = e / n, j = e - i * n;
    Ae[e] = -(S[e] + S[j * n + i]);
  }
  __syncthreads();
  const bool lmi = chol_copy(C, Ae, n, n);
  const bool pos = chol_copy(C, P, nbas, n);   // P(alpha): the top-left nbas x nbas corner
  if (threadIdx.x == 0 && !(lmi && pos)) atomicAdd(nfail, 1);
}

// Diagonal of the Schur complement, dense (K x K) or tiled (diagonal pair tiles, Ntil x Ntil):
// element q of the diagonal sits at G + q*(K+1) (dense) or tile(h,h) + s*(Ntil+1), q = h*Ntil + s.
__device__ __forceinline__ int64_t diag_off(int64_t q, int64_t K, int64_t Ntil, int64_t L0, int tiled) {
  if (!tiled) return q * (K + 1);
  const int64_t h = q / Ntil, s = q - h * Ntil;
  const int64_t p = h * L0 - h * (h - 1) / 2;   // pair index of (h, h)
  return p * Ntil * Ntil + s * (Ntil + 1);
}
__global__ void k_diag_sum(const double* __restrict__ G, int64_t K, int64_t Ntil, int64_t L0, int tiled,
                           double* __restrict__ part) {
  __shared__ double red[256];
  double acc = 0.0;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < K; q += (int64_t)gridDim.x * blockDim.x)
    acc += G[diag_off(q, K, Ntil, L0, tiled)];
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}
__global__ void k_diag_shift(double* __restrict__ G, int64_t K, int64_t Ntil, int64_t L0, int tiled, double shift) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < K; q += (int64_t)gridDim.x * blockDim.x)
    G[diag_off(q, K, Ntil, L0, tiled)] += shift;
}

constexpr int64_t kSolveNB = 1024;   // row panels of the dense triangular solves (dense_potrs)

struct Ipm {
  int64_t nb = 0, n = 0, K = 0;
  double *W = nullptr, *Rd = nullptr, *T1 = nullptr, *T2 = nullptr, *dX1 = nullptr, *dZ1 = nullptr, *dX2 = nullptr,
         *dZ2 = nullptr, *G = nullptr, *O1 = nullptr, *O2 = nullptr, *dy1 = nullptr, *dy2 = nullptr, *tmpK = nullptr,
         *tb = nullptr, *part = nullptr, *dc = nullptr, *work = nullptr;
  int* info = nullptr;
  int* fail = nullptr;
  int lwork = 0;
  bool tiled = false;          // G held as pair tiles (lower block triangle in column-major view)
  bool dist = false;           // SHARD_CYCLIC: this rank's pair tiles only, factorised across the ranks
  double* panel[2] = {};       // dist, nranks > 1: the broadcast panel of step k ((L0-1) tiles), by k parity
  double* lkk[2] = {};         // dist, nranks > 1: the broadcast diagonal factor L_kk (one tile), by k parity
  double* stat = nullptr;      // dist: {local error, potrf info} of a step, max-reduced over the ranks
  double *S1 = nullptr, *S2 = nullptr, *S3 = nullptr, *tb2 = nullptr;   // step_lens: the second chain's scratch
  cudaStream_t sl = nullptr;                  // step_lens: the second chain's stream
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  double* dinv = nullptr;      // dense: inverses of the kSolveNB diagonal blocks of the factor
  double* eye = nullptr;       // dense: nblk identity blocks (the right-hand side of those trsm)
  double* tsol = nullptr;      // dense: one block of the solve
  const double** dptrA = nullptr;   // dense: device pointers of the diagonal blocks (batched trsm)
  double** dptrB = nullptr;
  cusolverDnHandle_t sol = nullptr;
  cublasHandle_t blas = nullptr;
  cublasHandle_t blas_upd = nullptr;   // dist: the trailing update's handle (own workspace), on `upd`
  cudaStream_t upd = nullptr;          // dist: look-ahead stream of the trailing updates
  std::vector<cudaEvent_t> ev_pan, ev_col, ev_upd;   // dist: per step (panel solved / column k+1 / update done)
  cudaEvent_t ev[6] = {};
};

constexpr int kScalarBlocks = 256;

}  // namespace
}  // namespace polya

using namespace polya;

void polya_ipm_free(polya::Ctx& c) {
  Ipm* w = (Ipm*)c.ipm;
  if (!w) return;
  double* ps[] = {w->W, w->Rd, w->T1, w->T2, w->dX1, w->dZ1, w->dX2, w->dZ2, w->G, w->O1, w->O2,
                  w->dy1, w->dy2, w->tmpK, w->tb, w->part, w->dc, w->work, w->panel[0], w->panel[1],
                  w->lkk[0], w->lkk[1], w->stat, w->dinv, w->eye, w->tsol, w->S1, w->S2, w->S3, w->tb2};
  for (double* p : ps)
    if (p) cudaFree(p);
  if (w->info) cudaFree(w->info);
  if (w->fail) cudaFree(w->fail);
  if (w->dptrA) cudaFree((void*)w->dptrA);
  if (w->dptrB) cudaFree(w->dptrB);
  if (w->sol) cusolverDnDestroy(w->sol);
  if (w->blas) cublasDestroy(w->blas);
  if (w->blas_upd) cublasDestroy(w->blas_upd);
  if (w->upd) cudaStreamDestroy(w->upd);
  if (w->sl) cudaStreamDestroy(w->sl);
  if (w->ev_fork) cudaEventDestroy(w->ev_fork);
  if (w->ev_join) cudaEventDestroy(w->ev_join);
  for (auto* v : {&w->ev_pan, &w->ev_col, &w->ev_upd})
    for (auto e : *v) cudaEventDestroy(e);
  for (auto& e : w->ev)
    if (e) cudaEventDestroy(e);
  delete w;
  c.ipm = nullptr;
}

namespace {

struct IpmFail {
  polya_status s;
  std::string msg;
};
#define CK(x)                                                                                      \
  do {                                                                                             \
    cudaError_t e_ = (x);                                                                          \
    if (e_ != cudaSuccess) throw IpmFail{e_ == cudaErrorMemoryAllocation ? POLYA_ENOMEM : POLYA_ECUDA, \
                                         std::string(#x) + ": " + cudaGetErrorString(e_)};         \
  } while (0)
#define CB(x)                                                                                      \
  do {                                                                                             \
    cublasStatus_t e_ = (x);                                                                       \
    if (e_ != CUBLAS_STATUS_SUCCESS) throw IpmFail{POLYA_ECUDA, std::string(#x) + " failed"};      \
  } while (0)
#define CS(x)                                                                                      \
  do {                                                                                             \
    cusolverStatus_t e_ = (x);                                                                     \
    if (e_ != CUSOLVER_STATUS_SUCCESS) throw IpmFail{POLYA_ECUDA, std::string(#x) + " failed"};    \
  } while (0)

bool want_tiled(const Ctx& c) {
  if (c.cfg.shard == POLYA_SHARD_CYCLIC) return true;   // the distributed factorisation works on tiles
  if (c.fact_mode == 1) return false;
  if (c.fact_mode == 2) return true;
  size_t fr = 0, tot = 0;
  if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) return false;
  return (double)c.K * (double)c.K * 8.0 > 0.45 * (double)tot;   // the dense K x K G would not fit comfortably
}

Ipm* ipm_ws(Ctx& c) {
  if (c.ipm && ((Ipm*)c.ipm)->tiled != want_tiled(c)) polya_ipm_free(c);   // factorisation mode changed
  if (c.ipm) return (Ipm*)c.ipm;
  Ipm* w = new Ipm();
  c.ipm = w;
  w->nb = c.nb; w->n = c.n; w->K = c.K;
  w->tiled = want_tiled(c);
  const size_t st = (size_t)c.nb * c.n * c.n * sizeof(double), kv = (size_t)c.K * sizeof(double);
  double** stacks[] = {&w->W, &w->Rd, &w->T1, &w->T2, &w->dX1, &w->dZ1, &w->dX2, &w->dZ2, &w->S1, &w->S2, &w->S3};
  for (double** p : stacks) CK(cudaMalloc(p, st));
  double** vecs[] = {&w->O1, &w->O2, &w->dy1, &w->dy2, &w->tmpK};
  for (double** p : vecs) CK(cudaMalloc(p, kv));
  w->dist = c.cfg.shard == POLYA_SHARD_CYCLIC;
  CK(cudaMalloc(&w->G, (w->tiled ? (size_t)std::max<int64_t>(c.npairs_local, 1) * c.Ntil * c.Ntil : (size_t)c.K * c.K) *
                           sizeof(double)));
  if (w->dist && c.cfg.nranks > 1 && c.L0 > 1)
    for (int q = 0; q < 2; ++q) {
      CK(cudaMalloc(&w->panel[q], (size_t)(c.L0 - 1) * c.Ntil * c.Ntil * sizeof(double)));
      CK(cudaMalloc(&w->lkk[q], (size_t)c.Ntil * c.Ntil * sizeof(double)));
    }
  if (w->dist) {
    CK(cudaMalloc(&w->stat, 2 * sizeof(double)));
    CK(cudaStreamCreateWithFlags(&w->upd, cudaStreamNonBlocking));
    for (auto* v : {&w->ev_pan, &w->ev_col, &w->ev_upd}) {
      v->resize(c.L0 + 1);
      for (auto& e : *v) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
  }
  if (!w->tiled) {   // dense_potrs: diagonal-block inverses (~ K x kSolveNB doubles: 0.4 GB at config 4)
    const int64_t NB = kSolveNB, nblk = (c.K + NB - 1) / NB;
    CK(cudaMalloc(&w->dinv, (size_t)(nblk * NB * NB) * sizeof(double)));
    CK(cudaMalloc(&w->eye, (size_t)(nblk * NB * NB) * sizeof(double)));
    CK(cudaMalloc(&w->tsol, (size_t)NB * sizeof(double)));
    std::vector<double> I((size_t)(NB * NB), 0.0);
    for (int64_t q = 0; q < NB; ++q) I[(size_t)(q * NB + q)] = 1.0;
    for (int64_t b = 0; b < nblk; ++b)
      CK(cudaMemcpy(w->eye + b * NB * NB, I.data(), I.size() * sizeof(double), cudaMemcpyHostToDevice));
    std::vector<const double*> pa(nblk);
    std::vector<double*> pb(nblk);
    for (int64_t b = 0; b < nblk; ++b) {
      pa[b] = w->G + b * NB * c.K + b * NB;
      pb[b] = w->dinv + b * NB * NB;
    }
    CK(cudaMalloc((void**)&w->dptrA, nblk * sizeof(double*)));
    CK(cudaMalloc((void**)&w->dptrB, nblk * sizeof(double*)));
    CK(cudaMemcpy((void*)w->dptrA, pa.data(), nblk * sizeof(double*), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(w->dptrB, pb.data(), nblk * sizeof(double*), cudaMemcpyHostToDevice));
  }
  CK(cudaMalloc(&w->tb, (size_t)c.nb * sizeof(double)));
  CK(cudaMalloc(&w->tb2, (size_t)c.nb * sizeof(double)));
  CK(cudaStreamCreateWithFlags(&w->sl, cudaStreamNonBlocking));
  CK(cudaEventCreateWithFlags(&w->ev_fork, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&w->ev_join, cudaEventDisableTiming));
  CK(cudaMalloc(&w->part, (size_t)kScalarBlocks * 3 * sizeof(double)));
  CK(cudaMalloc(&w->dc, (size_t)std::max<int64_t>(c.L, 1) * sizeof(double)));
  CK(cudaMemcpy(w->dc, c.c.data(), (size_t)c.L * sizeof(double), cudaMemcpyHostToDevice));
  CK(cudaMalloc(&w->info, sizeof(int)));
  CK(cudaMalloc(&w->fail, sizeof(int)));
  CS(cusolverDnCreate(&w->sol));
  const int fdim = (int)(w->tiled ? c.Ntil : c.K);
  CS(cusolverDnDpotrf_bufferSize(w->sol, CUBLAS_FILL_MODE_LOWER, fdim, w->G, fdim, &w->lwork));
  CB(cublasCreate(&w->blas));
  if (w->dist) CB(cublasCreate(&w->blas_upd));
  CK(cudaMalloc(&w->work, (size_t)std::max(w->lwork, 1) * sizeof(double)));
  for (auto& e : w->ev) CK(cudaEventCreate(&e));
  return w;
}

void bgemm(Ctx& c, const double* A, int ta, const double* B, int tb, double* C, double alpha, double beta,
           cudaStream_t s) {
  const int tiles = (int)((c.n + 31) / 32);
  dim3 grid((unsigned)(tiles * tiles), (unsigned)c.nb);
  k_bgemm<<<grid, 128, 0, s>>>((int)c.n, A, ta, B, tb, C, alpha, beta, tiles);
  ++c.launches;
  CK(cudaGetLastError());
}

void axpby(Ctx& c, double a, const double* X, double b, const double* Y, double* out, const double* cdiag, double cs,
           cudaStream_t s) {
  const int64_t total = c.nb * c.n * c.n;
  k_axpby<<<(unsigned)std::min<int64_t>((total + 255) / 256, 4096), 256, 0, s>>>(total, (int)c.n, (int)c.nbas, c.L, a, X, b, Y, out,
                                                                                 cdiag, cs, c.d_CL);
  ++c.launches;
  CK(cudaGetLastError());
}

void sym(Ctx& c, const double* M, double* out, cudaStream_t s) {
  k_sym<<<(unsigned)c.nb, 256, 0, s>>>((int)c.n, M, out);
  ++c.launches;
  CK(cudaGetLastError());
}

void vaxpby(Ctx& c, double a, const double* x, double b, const double* y, double* out, cudaStream_t s) {
  k_vec_axpby<<<(unsigned)std::min<int64_t>((c.K + 255) / 256, 4096), 256, 0, s>>>(c.K, a, x, b, y, out);
  ++c.launches;
  CK(cudaGetLastError());
}

// Reading R5: t = min(1, 0.98 t_max), t_max = min_b 1 / max(0, -lambda_min(L_b^{-1} dS_b L_b^{-T})).
// Scratch: T1 (L^{-1}), T2 (L^{-1} dS), dX2 (M) -- free at this point of the step.
// One chain of reading R5 on stream st: L^{-1} (k_block_inv), M = L^{-1} dS L^{-T} (two k_bgemm into the
// scratch stacks Ta, Tb, M), per-block bound tb (k_block_lmin).
void step_chain(Ctx& c, const double* S, const double* dS, double* Ta, double* Tb, double* M, double* tb, double tcap,
                cudaStream_t st) {
  k_block_inv<<<(unsigned)c.nb, 512, block_inv_smem(c.n), st>>>((int)c.n, S, Ta, nullptr, 1);
  ++c.launches;
  CK(cudaGetLastError());
  bgemm(c, Ta, 0, dS, 0, Tb, 1.0, 0.0, st);   // L^{-1} dS
  bgemm(c, Tb, 0, Ta, 1, M, 1.0, 0.0, st);    // M = L^{-1} dS L^{-T}
  k_block_lmin<<<(unsigned)c.nb, 512, block_lmin_smem(c.n), st>>>((int)c.n, M, tcap, tb);
  ++c.launches;
  CK(cudaGetLastError());
}

// Reading R5 for both step lengths: t_p from (X, dX) and t_d from (Z, dZ), t = min(1, 0.98 t_max), t_max =
// min_b 1 / max(0, -lambda_min(L_b^{-1} dS_b L_b^{-T})).  The two chains are independent and each fills
// only ~70 % of the SM slots with latency-bound CTAs, so the second runs on w->sl (own scratch) beside the
// first; one host synchronisation for both.  Scratch of the first: T1, T2, dX2 (free at this point).
void step_lens(Ctx& c, Ipm* w, const double* X, const double* dX, const double* Z, const double* dZ, cudaStream_t s,
               double& tp, double& td) {
  const double frac = 0.98, tcap = 1.0 / frac;
  CK(cudaFuncSetAttribute(k_block_inv, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)block_inv_smem(c.n)));
  CK(cudaFuncSetAttribute(k_block_lmin, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)block_lmin_smem(c.n)));
  CK(cudaEventRecord(w->ev_fork, s));
  CK(cudaStreamWaitEvent(w->sl, w->ev_fork, 0));
  step_chain(c, X, dX, w->T1, w->T2, w->dX2, w->tb, tcap, s);
  step_chain(c, Z, dZ, w->S1, w->S2, w->S3, w->tb2, tcap, w->sl);
  CK(cudaEventRecord(w->ev_join, w->sl));
  CK(cudaStreamWaitEvent(s, w->ev_join, 0));
  std::vector<double> tb(2 * c.nb);
  CK(cudaMemcpyAsync(tb.data(), w->tb, c.nb * sizeof(double), cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(tb.data() + c.nb, w->tb2, c.nb * sizeof(double), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  double t[2];
  for (int q = 0; q < 2; ++q) {
    double* h = tb.data() + q * c.nb;
    if (*std::min_element(h, h + c.nb) < 0.0) {   // a semidefinite S_b: bisection for those blocks
      const double* S = q ? Z : X;
      const double* dS = q ? dZ : dX;
      double* d = q ? w->tb2 : w->tb;
      const size_t smb = (size_t)c.n * c.n * sizeof(double);
      CK(cudaFuncSetAttribute(k_block_tmax, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smb));
      k_block_tmax<<<(unsigned)c.nb, 256, smb, s>>>((int)c.n, S, dS, tcap, d);
      ++c.launches;
      CK(cudaGetLastError());
      CK(cudaMemcpyAsync(h, d, c.nb * sizeof(double), cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
    }
    double m = tcap;
    for (int64_t i = 0; i < c.nb; ++i) m = std::min(m, h[i]);
    t[q] = std::min(1.0, frac * m);
  }
  tp = t[0];
  td = t[1];
}

// ---- blocked Cholesky on the pair tiles --------------------------------------------------------
// Tile of pair (h <= h') holds G[h-block][h'-block] row-major = the block B_{h'h} of the LOWER block
// triangle in column-major view (N = Ntil).  G = L L^T, right-looking, L overwriting B.
// The tiles are this rank's pairs in pair order (all pairs on one rank; SHARD_CYCLIC: pair rows
// h = rank mod nranks), so the local index comes from the set-up's pair_local table.
inline double* tile(const Ctx& c, double* G, int64_t h, int64_t h2) {
  const int64_t p = h * c.L0 - h * (h - 1) / 2 + (h2 - h);
  return G + (int64_t)c.pair_local[p] * c.Ntil * c.Ntil;
}
inline double* tile(const Ctx& c, Ipm* w, int64_t h, int64_t h2) { return tile(c, w->G, h, h2); }

void tiled_potrf(Ctx& c, Ipm* w, cudaStream_t s) {
  const int N = (int)c.Ntil;
  const int64_t T = c.L0;
  const double one = 1.0, mone = -1.0;
  CB(cublasSetStream(w->blas, s));
  CK(cudaMemsetAsync(w->info, 0, sizeof(int), s));
  for (int64_t k = 0; k < T; ++k) {
    double* Lkk = tile(c, w, k, k);
    CS(cusolverDnDpotrf(w->sol, CUBLAS_FILL_MODE_LOWER, N, Lkk, N, w->work, w->lwork, w->info));
    int hinfo = 0;
    CK(cudaMemcpyAsync(&hinfo, w->info, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (hinfo != 0)
      throw IpmFail{POLYA_ENOTPD, "Schur complement not positive definite (tile " + std::to_string(k) + ", info " +
                                      std::to_string(hinfo) + ")"};
    for (int64_t i = k + 1; i < T; ++i)   // B_ik <- B_ik L_kk^{-T}
      CB(cublasDtrsm(w->blas, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T, CUBLAS_DIAG_NON_UNIT, N, N, &one,
                     Lkk, N, tile(c, w, k, i), N));
    for (int64_t i = k + 1; i < T; ++i) {  // trailing update B_ij -= B_ik B_jk^T, k < j <= i
      const double* Bik = tile(c, w, k, i);
      CB(cublasDsyrk(w->blas, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, N, N, &mone, Bik, N, &one, tile(c, w, i, i), N));
      for (int64_t j = k + 1; j < i; ++j)
        CB(cublasDgemm(w->blas, CUBLAS_OP_N, CUBLAS_OP_T, N, N, N, &mone, Bik, N, tile(c, w, k, j), N, &one,
                       tile(c, w, j, i), N));
    }
  }
  c.launches += T * (T + 1) * (T + 2) / 6 + T * (T + 1) / 2;
}

// x <- G^{-1} x with the tiled factor: L z = x (forward), L^T x = z (backward).
void tiled_potrs(Ctx& c, Ipm* w, double* x, cudaStream_t s) {
  const int N = (int)c.Ntil;
  const int64_t T = c.L0;
  const double one = 1.0, mone = -1.0;
  CB(cublasSetStream(w->blas, s));
  for (int64_t k = 0; k < T; ++k) {
    double* xk = x + k * N;
    CB(cublasDtrsv(w->blas, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, N, tile(c, w, k, k), N, xk, 1));
    for (int64_t i = k + 1; i < T; ++i)
      CB(cublasDgemv(w->blas, CUBLAS_OP_N, N, N, &mone, tile(c, w, k, i), N, xk, 1, &one, x + i * N, 1));
  }
  for (int64_t k = T - 1; k >= 0; --k) {
    double* xk = x + k * N;
    for (int64_t i = k + 1; i < T; ++i)
      CB(cublasDgemv(w->blas, CUBLAS_OP_T, N, N, &mone, tile(c, w, k, i), N, x + i * N, 1, &one, xk, 1));
    CB(cublasDtrsv(w->blas, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T, CUBLAS_DIAG_NON_UNIT, N, tile(c, w, k, k), N, xk, 1));
  }
  c.launches += 2 * T * (T + 1) / 2 + 2 * T;
}

// ---- distributed blocked Cholesky (SHARD_CYCLIC) -------------
// Block column k of the lower factor is pair row k (tiles (k, i), i >= k), held by rank k mod N
// (column-cyclic: the trailing-update work sum_{j = r mod N} j (L0 - j) is balanced to a few %).
// Step k: the owner factors L_kk and broadcasts it with the raw panel B_ik (i > k, contiguous in
// its pair order); the ranks split the panel solves B_ik <- B_ik L_kk^{-T} (tile q = i-k-1 on rank
// q mod N: one rank doing all of them would put ~3.6 s of serial trsm on config 5's critical path)
// and broadcast the solved tiles back; every rank then updates its own block columns j > k,
// B_ij -= B_ik B_jk^T (k < j <= i).  Each tile sees the same cuBLAS / cuSOLVER calls in the same
// order as in tiled_potrf, so the factor is the single-GPU one bit for bit.
inline int owner(const Ctx& c, int64_t k) { return (int)(k % c.cfg.nranks); }

int dist_potrf_kk(Ctx& c, Ipm* w, double* G, int64_t k, cudaStream_t s) {   // owner of column k only
  const int N = (int)c.Ntil;
  CS(cusolverDnSetStream(w->sol, s));
  CS(cusolverDnDpotrf(w->sol, CUBLAS_FILL_MODE_LOWER, N, tile(c, G, k, k), N, w->work, w->lwork, w->info));
  ++c.launches;
  int hinfo = 0;
  CK(cudaMemcpyAsync(&hinfo, w->info, sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return hinfo;
}

// This rank's share of the panel solve B_ik <- B_ik L_kk^{-T}: panel tiles q = i - k - 1 with
// q = rank mod nranks (all of them on one rank), in the rank's copy of the panel.
void dist_trsm_share(Ctx& c, Ipm* w, int64_t k, const double* Lkk, double* panel, cudaStream_t s) {
  const int N = (int)c.Ntil;
  const int64_t NN = (int64_t)N * N;
  const double one = 1.0;
  CB(cublasSetStream(w->blas, s));
  for (int64_t q = c.cfg.rank; q < c.L0 - k - 1; q += c.cfg.nranks) {
    CB(cublasDtrsm(w->blas, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T, CUBLAS_DIAG_NON_UNIT, N, N, &one,
                   Lkk, N, panel + q * NN, N));
    ++c.launches;
  }
}

// panel + (i - k - 1) N^2 = B_ik for i > k; this rank's block columns j in [j0, j1) (j > k)
void dist_update(Ctx& c, cublasHandle_t h, double* G, int64_t k, const double* panel, int64_t j0, int64_t j1,
                 cudaStream_t s) {
  const int N = (int)c.Ntil;
  const int64_t NN = (int64_t)N * N;
  const double one = 1.0, mone = -1.0;
  CB(cublasSetStream(h, s));
  for (int64_t j = std::max(j0, k + 1); j < std::min(j1, c.L0); ++j) {
    if (owner(c, j) != c.cfg.rank) continue;
    const double* Bjk = panel + (j - k - 1) * NN;
    CB(cublasDsyrk(h, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, N, N, &mone, Bjk, N, &one, tile(c, G, j, j), N));
    ++c.launches;
    for (int64_t i = j + 1; i < c.L0; ++i) {
      CB(cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_T, N, N, N, &mone, panel + (i - k - 1) * NN, N, Bjk, N, &one,
                     tile(c, G, j, i), N));
      ++c.launches;
    }
  }
}

void comm(Ctx& c, cudaError_t e) {
  if (e == cudaErrorNotReady) throw IpmFail{POLYA_ENCCL, "distributed factorisation before polya_nccl_init"};
  if (e != cudaSuccess) throw IpmFail{POLYA_ENCCL, c.last_error};
}

// Collective agreement on a step's outcome: every rank contributes {its first local failure (a
// polya_status, 0 = none), the owner's potrf info}; the maxima come back to all ranks, so a failure on
// one rank makes every rank leave dist_potrf with the same error instead of waiting in a broadcast.
void dist_agree(Ctx& c, Ipm* w, polya_status& local, int& info, const std::string& msg, cudaStream_t s) {
  if (c.cfg.nranks == 1) {
    if (local != POLYA_OK) throw IpmFail{local, msg};
    return;
  }
  double h[2] = {(double)local, (double)info};
  CK(cudaMemcpyAsync(w->stat, h, sizeof(h), cudaMemcpyHostToDevice, s));
  comm(c, comm_allreduce_max(c, w->stat, 2, s));
  CK(cudaMemcpyAsync(h, w->stat, sizeof(h), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (h[0] != 0.0)
    throw IpmFail{(polya_status)(int)h[0], local != POLYA_OK ? msg : "distributed factorisation: a peer rank failed"};
  info = (int)h[1];
}

// Collective over the ranks of the context (NCCL, or the loopback group; nothing to send with one
// rank).  With look-ahead: the panel work of step k (the owner's potrf, the broadcasts, the split
// panel solves) runs on `s`, the trailing update on w->upd; the update of block column k+1 goes first
// and releases step k+1's panel (event), so the next panel factorisation and its broadcasts overlap the
// rest of step k's update.  Non-owners receive panels into two buffers by step parity (a buffer is
// reused only after the update of step k-2 has read it).  Every tile still sees the same calls in the
// same order as tiled_potrf: the factor is the one-rank factor bit for bit.
bool dist_potrf(Ctx& c, Ipm* w, double* G, cudaStream_t s) {
  const int64_t NN = c.Ntil * c.Ntil, T = c.L0;
  polya_status pending = POLYA_OK;   // a local failure not yet agreed on
  std::string pmsg;
  auto local = [&](auto&& f) {
    if (pending != POLYA_OK) return;
    try {
      f();
    } catch (const IpmFail& e) {
      pending = e.s;
      pmsg = e.msg;
    }
  };
  auto drain = [&]() { cudaStreamSynchronize(w->upd); };
  CK(cudaEventRecord(w->ev_col[0], s));   // G assembled (on s): the first panel may start
  CK(cudaStreamWaitEvent(w->upd, w->ev_col[0], 0));
  for (int64_t k = 0; k < T; ++k) {
    const int o = owner(c, k);
    const bool mine = c.cfg.rank == o;
    CK(cudaStreamWaitEvent(s, w->ev_col[k], 0));   // block column k fully updated by step k-1
    int info = 0;
    if (mine) local([&] { info = dist_potrf_kk(c, w, G, k, s); });
    try {
      dist_agree(c, w, pending, info, pmsg, s);
    } catch (...) {
      drain();
      throw;
    }
    if (info != 0) {
      drain();
      return false;
    }
    if (k + 1 == T) break;
    const int buf = (int)(k & 1);
    if (!mine && k >= 2) CK(cudaStreamWaitEvent(s, w->ev_upd[k - 2], 0));   // the buffer's last reader
    double* Lkk = mine ? tile(c, G, k, k) : w->lkk[buf];
    double* panel = mine ? tile(c, G, k, k + 1) : w->panel[buf];
    const int64_t nq = T - k - 1;
    comm(c, comm_bcast(c, Lkk, (size_t)NN, false, o, s));
    comm(c, comm_bcast(c, panel, (size_t)(nq * NN), false, o, s));
    local([&] { dist_trsm_share(c, w, k, Lkk, panel, s); });
    comm(c, comm_bcast_tiles(c, panel, (size_t)NN, nq, s));   // tile q from rank q mod N
    CK(cudaEventRecord(w->ev_pan[k], s));
    CK(cudaStreamWaitEvent(w->upd, w->ev_pan[k], 0));
    local([&] { dist_update(c, w->blas_upd, G, k, panel, k + 1, k + 2, w->upd); });   // column k+1 first
    CK(cudaEventRecord(w->ev_col[k + 1], w->upd));
    local([&] { dist_update(c, w->blas_upd, G, k, panel, k + 2, T, w->upd); });
    CK(cudaEventRecord(w->ev_upd[k], w->upd));
  }
  CK(cudaEventRecord(w->ev_upd[T], w->upd));
  CK(cudaStreamWaitEvent(s, w->ev_upd[T], 0));   // later work on s sees the whole factor
  int none = 0;
  dist_agree(c, w, pending, none, pmsg, s);
  return true;
}

// x <- G^{-1} x with the distributed factor: the owner of column k does its triangular solve and
// its panel's matrix-vector updates, then broadcasts the part of x it changed.
void dist_potrs(Ctx& c, Ipm* w, double* G, double* x, cudaStream_t s) {
  const int N = (int)c.Ntil;
  const int64_t T = c.L0;
  const double one = 1.0, mone = -1.0;
  CB(cublasSetStream(w->blas, s));
  for (int64_t k = 0; k < T; ++k) {
    const int o = owner(c, k);
    double* xk = x + k * N;
    if (c.cfg.rank == o) {
      CB(cublasDtrsv(w->blas, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, N, tile(c, G, k, k), N, xk, 1));
      for (int64_t i = k + 1; i < T; ++i)
        CB(cublasDgemv(w->blas, CUBLAS_OP_N, N, N, &mone, tile(c, G, k, i), N, xk, 1, &one, x + i * N, 1));
      c.launches += T - k;
    }
    comm(c, comm_bcast(c, xk, (size_t)((T - k) * N), false, o, s));
  }
  for (int64_t k = T - 1; k >= 0; --k) {
    const int o = owner(c, k);
    double* xk = x + k * N;
    if (c.cfg.rank == o) {
      for (int64_t i = k + 1; i < T; ++i)
        CB(cublasDgemv(w->blas, CUBLAS_OP_T, N, N, &mone, tile(c, G, k, i), N, x + i * N, 1, &one, xk, 1));
      CB(cublasDtrsv(w->blas, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T, CUBLAS_DIAG_NON_UNIT, N, tile(c, G, k, k), N, xk, 1));
      c.launches += T - k;
    }
    comm(c, comm_bcast(c, xk, (size_t)N, false, o, s));
  }
}

// G <- G + eps I, eps = 1e-12 tr(G) / K (the regularised retry) on this rank's diagonal tiles, the
// trace summed over the ranks.  Returns eps.
double dist_regularise(Ctx& c, Ipm* w, cudaStream_t s) {
  std::vector<double> part(kScalarBlocks);
  double tr = 0.0;
  for (int64_t h = 0; h < c.L0; ++h) {
    if (owner(c, h) != c.cfg.rank) continue;
    k_diag_sum<<<kScalarBlocks, 256, 0, s>>>(tile(c, w, h, h), c.Ntil, c.Ntil, 1, 1, w->part);
    ++c.launches;
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(part.data(), w->part, kScalarBlocks * sizeof(double), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    for (double v : part) tr += v;
  }
  CK(cudaMemcpyAsync(w->part, &tr, sizeof(double), cudaMemcpyHostToDevice, s));
  comm(c, comm_allreduce_sum(c, w->part, 1, s));
  CK(cudaMemcpyAsync(&tr, w->part, sizeof(double), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  const double eps = 1e-12 * std::fabs(tr) / (double)c.K;
  for (int64_t h = 0; h < c.L0; ++h) {
    if (owner(c, h) != c.cfg.rank) continue;
    k_diag_shift<<<kScalarBlocks, 256, 0, s>>>(tile(c, w, h, h), c.Ntil, c.Ntil, 1, 1, eps);
    ++c.launches;
    CK(cudaGetLastError());
  }
  return eps;
}

// x <- G^{-1} x with the dense factor (column-major lower L, leading dimension K), blocked by column
// panels of kSolveNB: forward t = L_kk^{-1} x_k, x_k = t, x_{k+1..} -= L_{k+1..,k} t; backward
// x_k -= L_{k+1..,k}^T x_{k+1..}, x_k = L_kk^{-T} x_k -- every step a gemv (the panel gemvs stream the
// factor once per pass; the diagonal inverses, formed once per factorisation by trsm against I, make
// the diagonal solves parallel).  cuSOLVER's dpotrs with one right-hand side is level-2 trsv, a chain
// of K/32 dependent 32-row steps: 10.8 ms per solve at config 4; a blocked variant that kept trsv on
// 4096-row diagonal blocks still spent 16.6 ms of a step in that chain.
void dense_potrs(Ctx& c, Ipm* w, double* x, cudaStream_t s) {
  const int64_t K = c.K, NB = kSolveNB, nblk = (K + NB - 1) / NB;
  const double one = 1.0, mone = -1.0, zero = 0.0;
  CB(cublasSetStream(w->blas, s));
  for (int64_t b = 0; b < nblk; ++b) {
    const int64_t k0 = b * NB;
    const int nb = (int)std::min<int64_t>(NB, K - k0), rest = (int)(K - k0 - nb);
    const double* Dinv = w->dinv + b * NB * NB;   // column-major nb x nb, ld NB
    CB(cublasDgemv(w->blas, CUBLAS_OP_N, nb, nb, &one, Dinv, (int)NB, x + k0, 1, &zero, w->tsol, 1));
    CK(cudaMemcpyAsync(x + k0, w->tsol, nb * sizeof(double), cudaMemcpyDeviceToDevice, s));
    if (rest > 0)
      CB(cublasDgemv(w->blas, CUBLAS_OP_N, rest, nb, &mone, w->G + k0 * K + k0 + nb, (int)K, x + k0, 1, &one,
                     x + k0 + nb, 1));
    c.launches += rest > 0 ? 2 : 1;
  }
  for (int64_t b = nblk - 1; b >= 0; --b) {
    const int64_t k0 = b * NB;
    const int nb = (int)std::min<int64_t>(NB, K - k0), rest = (int)(K - k0 - nb);
    const double* Dinv = w->dinv + b * NB * NB;
    if (rest > 0)
      CB(cublasDgemv(w->blas, CUBLAS_OP_T, rest, nb, &mone, w->G + k0 * K + k0 + nb, (int)K, x + k0 + nb, 1, &one,
                     x + k0, 1));
    CB(cublasDgemv(w->blas, CUBLAS_OP_T, nb, nb, &one, Dinv, (int)NB, x + k0, 1, &zero, w->tsol, 1));
    CK(cudaMemcpyAsync(x + k0, w->tsol, nb * sizeof(double), cudaMemcpyDeviceToDevice, s));
    c.launches += rest > 0 ? 2 : 1;
  }
}

// Inverses of the diagonal kSolveNB blocks of the dense factor (after a successful potrf): Dinv_b =
// L_bb^{-1} by trsm against the identity (column-major, ld NB; the strictly upper part is zero).
void dense_diag_inverses(Ctx& c, Ipm* w, cudaStream_t s) {
  const int64_t K = c.K, NB = kSolveNB, nblk = (K + NB - 1) / NB, full = K / NB;
  const double one = 1.0;
  CB(cublasSetStream(w->blas, s));
  CK(cudaMemcpyAsync(w->dinv, w->eye, (size_t)(nblk * NB * NB) * sizeof(double), cudaMemcpyDeviceToDevice, s));
  if (full > 0)   // the full blocks in one batched call (pointer arrays built with the workspace)
    CB(cublasDtrsmBatched(w->blas, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, (int)NB,
                          (int)NB, &one, w->dptrA, (int)K, w->dptrB, (int)NB, (int)full));
  if (full < nblk) {   // the ragged last block
    const int64_t k0 = full * NB;
    const int nb = (int)(K - k0);
    CB(cublasDtrsm(w->blas, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, nb, nb, &one,
                   w->G + k0 * K + k0, (int)K, w->dinv + full * NB * NB, (int)NB));
  }
  c.launches += 2;
}

void solveG(Ctx& c, Ipm* w, double* x, cudaStream_t s) {
  if (w->dist) dist_potrs(c, w, w->G, x, s);
  else if (w->tiled) tiled_potrs(c, w, x, s);
  else dense_potrs(c, w, x, s);
}

// Cholesky of the Schur complement (dense or tiled); false if not positive definite.
bool factor(Ctx& c, Ipm* w, cudaStream_t s) {
  if (w->dist) return dist_potrf(c, w, w->G, s);
  if (w->tiled) {
    try {
      tiled_potrf(c, w, s);
    } catch (const IpmFail& f) {
      if (f.s == POLYA_ENOTPD) return false;
      throw;
    }
    return true;
  }
  CS(cusolverDnDpotrf(w->sol, CUBLAS_FILL_MODE_LOWER, (int)c.K, w->G, (int)c.K, w->work, w->lwork, w->info));
  int hinfo = 0;
  CK(cudaMemcpyAsync(&hinfo, w->info, sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (hinfo != 0) return false;
  dense_diag_inverses(c, w, s);
  return true;
}

polya_status call(polya_status st, Ctx& c) {
  if (st != POLYA_OK) throw IpmFail{st, c.last_error};
  return st;
}

}  // namespace

extern "C" polya_status polya_ipm_step(polya_ctx* ctx, polya_ipm_state* st, polya_ipm_stats* stats, void* stream) {
  if (!ctx || !st || !st->X || !st->Z || !st->y) return POLYA_EINVAL;
  Ctx& c = ctx->c;
  if (c.cfg.nranks != 1 && c.cfg.shard != POLYA_SHARD_CYCLIC) {
    c.last_error = "polya_ipm_step on several ranks needs SHARD_CYCLIC (the distributed factorisation)";
    return POLYA_EINVAL;
  }
  if ((c.n * c.n + c.n) * (int64_t)sizeof(double) > 227 * 1024) {
    c.last_error = "polya_ipm_step: block too large for the shared-memory Cholesky (n <= 168)";
    return POLYA_EINVAL;
  }
  cudaStream_t s = (cudaStream_t)stream;
  double* X = st->X;
  double* Z = st->Z;
  double* y = st->y;
  const double mu = st->mu;
  try {
    Ipm* w = ipm_ws(c);
    CS(cusolverDnSetStream(w->sol, s));
    CK(cudaEventRecord(w->ev[0], s));
    // W = Z^-1
    CK(cudaMemsetAsync(w->fail, 0, sizeof(int), s));
    {
      const size_t smi = block_inv_smem(c.n);
      CK(cudaFuncSetAttribute(k_block_inv, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smi));
      k_block_inv<<<(unsigned)c.nb, 512, smi, s>>>((int)c.n, Z, w->W, w->fail);
      ++c.launches;
      CK(cudaGetLastError());
    }
    // Rd = -B^T(y) + Z + C
    call(polya_apply(ctx, y, w->T1, s), c);
    axpby(c, -1.0, w->T1, 1.0, Z, w->Rd, w->dc, 1.0, s);
    // O1 = B(W Rd X) - 1
    bgemm(c, w->Rd, 0, X, 0, w->T2, 1.0, 0.0, s);
    bgemm(c, w->W, 0, w->T2, 0, w->T1, 1.0, 0.0, s);
    call(polya_adjoint(ctx, w->T1, w->O1, s), c);
    k_vec_shift<<<(unsigned)std::min<int64_t>((c.K + 255) / 256, 4096), 256, 0, s>>>(c.K, -1.0, w->O1);  // - a
    ++c.launches;
    CK(cudaGetLastError());
    // G (FULL layout), then its Cholesky factor (timed separately)
    CK(cudaEventRecord(w->ev[1], s));
    const int glayout = w->tiled ? POLYA_G_PAIR_TILES : POLYA_G_FULL;
    call(polya_schur(ctx, X, w->W, w->G, glayout, s), c);
    CK(cudaEventRecord(w->ev[2], s));
    int hfail = 0;
    CK(cudaMemcpyAsync(&hfail, w->fail, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (hfail) throw IpmFail{POLYA_ENOTPD, "a Z block is not positive definite"};
    int retries = 0;
    if (!factor(c, w, s)) {
      // G near-singular (it becomes ill-conditioned near convergence): one retry on G + eps I with
      // eps = 1e-12 tr(G) / K (SURVEY 8(b) ENOTPD).  potrf destroyed G: re-assemble it.
      call(polya_schur(ctx, X, w->W, w->G, glayout, s), c);
      double eps = 0.0;
      if (w->dist) {
        eps = dist_regularise(c, w, s);
      } else {
        const int tiled = w->tiled ? 1 : 0;
        k_diag_sum<<<kScalarBlocks, 256, 0, s>>>(w->G, c.K, c.Ntil, c.L0, tiled, w->part);
        ++c.launches;
        CK(cudaGetLastError());
        std::vector<double> part(kScalarBlocks);
        CK(cudaMemcpyAsync(part.data(), w->part, kScalarBlocks * sizeof(double), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        double tr = 0.0;
        for (double v : part) tr += v;
        eps = 1e-12 * std::fabs(tr) / (double)c.K;
        k_diag_shift<<<kScalarBlocks, 256, 0, s>>>(w->G, c.K, c.Ntil, c.L0, tiled, eps);
        ++c.launches;
        CK(cudaGetLastError());
      }
      retries = 1;
      if (!(eps > 0.0) || !factor(c, w, s))
        throw IpmFail{POLYA_ENOTPD, "Schur complement not positive definite after one regularised retry"};
    }
    CK(cudaEventRecord(w->ev[3], s));
    // dy^ = G^-1 O1
    CK(cudaMemcpyAsync(w->dy1, w->O1, c.K * sizeof(double), cudaMemcpyDeviceToDevice, s));
    solveG(c, w, w->dy1, s);
    // dZ^ = -Rd + B^T(dy^);  dX^ = sym(-X + W (Rd - B^T(dy^)) X)
    call(polya_apply(ctx, w->dy1, w->T1, s), c);
    axpby(c, -1.0, w->Rd, 1.0, w->T1, w->dZ1, nullptr, 0.0, s);          // dZ^
    axpby(c, 1.0, w->Rd, -1.0, w->T1, w->T2, nullptr, 0.0, s);           // Rd - B^T(dy^)
    bgemm(c, w->T2, 0, X, 0, w->T1, 1.0, 0.0, s);                          // (Rd - B^T dy^) X
    bgemm(c, w->W, 0, w->T1, 0, w->T2, 1.0, 0.0, s);                       // W (...) X
    axpby(c, -1.0, X, 1.0, w->T2, w->T1, nullptr, 0.0, s);                 // -X + W (...) X
    sym(c, w->T1, w->dX1, s);
    // O2 = mu B(W) - B(W dZ^ dX^);  dy- = G^-1 O2
    bgemm(c, w->dZ1, 0, w->dX1, 0, w->T1, 1.0, 0.0, s);                    // dZ^ dX^
    bgemm(c, w->W, 0, w->T1, 0, w->T2, 1.0, 0.0, s);                       // W dZ^ dX^  (kept in T2)
    call(polya_adjoint(ctx, w->W, w->tmpK, s), c);
    call(polya_adjoint(ctx, w->T2, w->O2, s), c);
    vaxpby(c, mu, w->tmpK, -1.0, w->O2, w->O2, s);
    CK(cudaMemcpyAsync(w->dy2, w->O2, c.K * sizeof(double), cudaMemcpyDeviceToDevice, s));
    solveG(c, w, w->dy2, s);
    // dZ- = B^T(dy-);  dX- = sym(mu W - W dZ^ dX^ - W dZ- X)
    call(polya_apply(ctx, w->dy2, w->dZ2, s), c);
    bgemm(c, w->dZ2, 0, X, 0, w->T1, 1.0, 0.0, s);                         // dZ- X
    bgemm(c, w->W, 0, w->T1, 0, w->T2, -1.0, -1.0, s);                     // T2 = -W dZ^ dX^ - W dZ- X
    axpby(c, mu, w->W, 1.0, w->T2, w->T1, nullptr, 0.0, s);
    sym(c, w->T1, w->dX2, s);
    // totals (into dX1, dZ1, dy1)
    axpby(c, 1.0, w->dX1, 1.0, w->dX2, w->dX1, nullptr, 0.0, s);
    axpby(c, 1.0, w->dZ1, 1.0, w->dZ2, w->dZ1, nullptr, 0.0, s);
    vaxpby(c, 1.0, w->dy1, 1.0, w->dy2, w->dy1, s);
    // line search (R5) and update (R6)
    double tp = 0.0, td = 0.0;
    step_lens(c, w, X, w->dX1, Z, w->dZ1, s, tp, td);
    if (!(tp > 0.0) || !(td > 0.0)) throw IpmFail{POLYA_ESTEP, "no admissible step"};
    axpby(c, 1.0, X, tp, w->dX1, X, nullptr, 0.0, s);
    axpby(c, 1.0, Z, td, w->dZ1, Z, nullptr, 0.0, s);
    vaxpby(c, 1.0, y, td, w->dy1, y, s);
    // step 4 scalars
    const int64_t total = c.nb * c.n * c.n;
    k_scalars<<<kScalarBlocks, 256, 0, s>>>(total, (int)c.n, (int)c.nbas, c.L, Z, X, w->dc, y, c.K, w->part, c.d_CL);
    ++c.launches;
    CK(cudaGetLastError());
    std::vector<double> part(kScalarBlocks * 3);
    CK(cudaMemcpyAsync(part.data(), w->part, part.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
    CK(cudaEventRecord(w->ev[4], s));
    CK(cudaStreamSynchronize(s));
    double trzx = 0, phi = 0, psi = 0;
    for (int b = 0; b < kScalarBlocks; ++b) { trzx += part[b * 3]; phi += part[b * 3 + 1]; psi += part[b * 3 + 2]; }
    const double mu_new = trzx / (3.0 * (double)c.nb * (double)c.n);
    st->mu = mu_new;
    st->iter += 1;
    if (stats) {
      stats->gap = std::fabs(phi - psi);
      stats->mu = mu_new;
      stats->tp = tp;
      stats->td = td;
      stats->phi = phi;
      stats->psi = psi;
      float a = 0, b = 0, tot = 0;
      cudaEventElapsedTime(&a, w->ev[1], w->ev[2]);
      cudaEventElapsedTime(&b, w->ev[2], w->ev[3]);
      cudaEventElapsedTime(&tot, w->ev[0], w->ev[4]);
      stats->ms_schur = a;
      stats->ms_factor = b;
      stats->ms_other = tot - a - b;
      stats->reg_retries = retries;
    }
  } catch (const IpmFail& f) {
    c.last_error = f.msg;
    return f.s;
  }
  return POLYA_OK;
}

// ---- test hook: the IPM's blockwise kernels on caller-given block stacks -----------------------
// W = S^{-1} (k_block_inv), L^{-1} (k_block_inv, L^{-1} mode), M = L^{-1} dS L^{-T} (two k_bgemm) and
// t_b = min(1/0.98, 1/max(0, -lambda_min(M_b))) (k_block_lmin) -- the kernels step_len and the W of
// polya_ipm_step run, at any block order n <= 168, so their parity and the maximum size are tested
// directly (tests/test_gpu_block_kernels.py).
extern "C" polya_status polya_block_kernels_test(int32_t n, int64_t nb, const double* S, const double* dS, double* W,
                                                 double* Linv, double* M, double* t, int32_t* fail, void* stream) {
  if (n < 1 || n > 168 || nb < 1 || !S || !dS || !W || !Linv || !M || !t || !fail) return POLYA_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  double* T = nullptr;
  auto ck = [&](cudaError_t e) {
    if (e != cudaSuccess) throw IpmFail{POLYA_ECUDA, cudaGetErrorString(e)};
  };
  try {
    const size_t nbytes = (size_t)nb * n * n * sizeof(double);
    ck(cudaMalloc(&T, nbytes));
    ck(cudaMemsetAsync(fail, 0, sizeof(int32_t), s));
    const size_t smi = block_inv_smem(n), sml = block_lmin_smem(n);
    ck(cudaFuncSetAttribute(k_block_inv, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smi));
    ck(cudaFuncSetAttribute(k_block_lmin, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sml));
    k_block_inv<<<(unsigned)nb, 512, smi, s>>>(n, S, W, fail);
    k_block_inv<<<(unsigned)nb, 512, smi, s>>>(n, S, Linv, nullptr, 1);
    const int tiles = (n + 31) / 32;
    dim3 grid((unsigned)(tiles * tiles), (unsigned)nb);
    k_bgemm<<<grid, 128, 0, s>>>(n, Linv, 0, dS, 0, T, 1.0, 0.0, tiles);   // L^{-1} dS
    k_bgemm<<<grid, 128, 0, s>>>(n, T, 0, Linv, 1, M, 1.0, 0.0, tiles);    // (L^{-1} dS) L^{-T}
    k_block_lmin<<<(unsigned)nb, 512, sml, s>>>(n, M, 1.0 / 0.98, t);
    ck(cudaGetLastError());
    ck(cudaStreamSynchronize(s));
    ck(cudaFree(T));
  } catch (const IpmFail& f) {
    if (T) cudaFree(T);
    return f.s;
  }
  return POLYA_OK;
}

// ---- the distributed factorisation with an in-process loopback in place of NCCL (tests) --------
// All ranks' contexts live in this process on one device; each rank is a host thread with its own
// stream running the SAME dist_potrf / dist_potrs as the NCCL path, the collectives going through the
// loopback group (combine.cpp: barrier + device copies from the root's buffer) instead of NCCL.  This
// checks the partition, the local tile indexing, the panel bookkeeping, the look-ahead ordering and the
// x exchange of the multi-rank path on one GPU (NCCL refuses two ranks on one device).  x (K doubles):
// b in, G^{-1} b out (every rank's copy is the same; rank 0's is returned).
extern "C" polya_status polya_factor_solve_loopback(polya_ctx** ctxs, int32_t nranks, double* const* G_local, double* x,
                                                    void* stream) {
  if (!ctxs || nranks < 1 || !G_local || !x) return POLYA_EINVAL;
  for (int32_t r = 0; r < nranks; ++r) {
    if (!ctxs[r] || !G_local[r]) return POLYA_EINVAL;
    const Ctx& c = ctxs[r]->c;
    if (c.cfg.shard != POLYA_SHARD_CYCLIC || c.cfg.nranks != nranks || c.cfg.rank != r || c.K != ctxs[0]->c.K ||
        c.nccl)
      return POLYA_EINVAL;
  }
  cudaStream_t s0 = (cudaStream_t)stream;
  Ctx& c0 = ctxs[0]->c;
  if (cudaStreamSynchronize(s0) != cudaSuccess) return POLYA_ECUDA;   // G_local and x are ready
  LoopGroup g;
  g.n = nranks;
  g.ptr.assign(nranks, nullptr);
  g.host.resize(nranks);
  std::vector<polya_status> st(nranks, POLYA_OK);
  std::vector<std::string> msg(nranks);
  std::vector<std::thread> th;
  for (int32_t r = 0; r < nranks; ++r) ctxs[r]->c.loop = &g;
  for (int32_t r = 0; r < nranks; ++r)
    th.emplace_back([&, r] {
      Ctx& c = ctxs[r]->c;
      cudaStream_t s = nullptr;
      try {
        CK(cudaSetDevice(c.device));
        CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        Ipm* w = ipm_ws(c);
        CK(cudaMemcpyAsync(w->tmpK, x, c.K * sizeof(double), cudaMemcpyDeviceToDevice, s));
        if (!dist_potrf(c, w, G_local[r], s))
          throw IpmFail{POLYA_ENOTPD, "Schur complement not positive definite"};
        dist_potrs(c, w, G_local[r], w->tmpK, s);
        CK(cudaStreamSynchronize(s));
      } catch (const IpmFail& f) {
        st[r] = f.s;
        msg[r] = f.msg;
        loop_abort(&g);
      }
      if (s) cudaStreamDestroy(s);
    });
  for (auto& t : th) t.join();
  for (int32_t r = 0; r < nranks; ++r) ctxs[r]->c.loop = nullptr;
  for (int32_t r = 0; r < nranks; ++r)   // the root cause first: an aborted peer reports ENCCL
    if (st[r] != POLYA_OK && st[r] != POLYA_ENCCL) {
      c0.last_error = msg[r];
      return st[r];
    }
  for (int32_t r = 0; r < nranks; ++r)
    if (st[r] != POLYA_OK) {
      c0.last_error = msg[r];
      return st[r];
    }
  Ipm* w0 = (Ipm*)c0.ipm;
  if (cudaMemcpyAsync(x, w0->tmpK, c0.K * sizeof(double), cudaMemcpyDeviceToDevice, s0) != cudaSuccess ||
      cudaStreamSynchronize(s0) != cudaSuccess)
    return POLYA_ECUDA;
  return POLYA_OK;
}

// ---- Algorithm 2 to its stopping rule, and the verdict ---------------------

extern "C" polya_status polya_ipm_solve(polya_ctx* ctx, polya_ipm_state* st, const polya_solve_opts* opt,
                                        polya_solve_result* res, void* stream) {
  if (!ctx || !st || !st->X || !st->Z || !st->y || !opt || !res) return POLYA_EINVAL;
  Ctx& c = ctx->c;
  cudaStream_t s = (cudaStream_t)stream;
  std::memset(res, 0, sizeof(*res));
  res->status = POLYA_EMAXIT;
  try {
    if (opt->init) {   // X = Z = I, y = 0, mu = tr(ZX) / (3 (L+M) n) = 1/3 (R4)
      const int64_t total = c.nb * c.n * c.n;
      k_identity<<<(unsigned)std::min<int64_t>((total + 255) / 256, 4096), 256, 0, s>>>(total, (int)c.n, st->X, st->Z);
      ++c.launches;
      CK(cudaGetLastError());
      CK(cudaMemsetAsync(st->y, 0, (size_t)c.K * sizeof(double), s));
      st->mu = 1.0 / 3.0;
      st->iter = 0;
    }
    std::vector<double> part(kScalarBlocks);
    for (int it = 0; it < opt->maxit; ++it) {
      polya_ipm_stats ps;
      std::memset(&ps, 0, sizeof(ps));
      const polya_status r = polya_ipm_step(ctx, st, &ps, stream);
      res->iterations = it + 1;
      if (opt->history) opt->history[it] = ps;
      if (r == POLYA_ENOTPD || r == POLYA_ESTEP) {   // an outcome, not an exception
        res->status = r;
        return POLYA_OK;
      }
      if (r != POLYA_OK) return r;   // misuse, allocation, CUDA or NCCL failure: the caller's error
      if (!std::isfinite(ps.phi) || !std::isfinite(ps.psi) || !std::isfinite(ps.mu) ||
          std::max(std::fabs(ps.phi), std::max(std::fabs(ps.psi), ps.mu)) > POLYA_DIVERGENCE_BOUND) {
        res->gap = ps.gap;   // reading R20: an unbounded iterate, the LMI is infeasible
        res->mu = ps.mu;
        res->status = POLYA_EDIVERGED;
        return POLYA_OK;
      }
      res->gap = ps.gap;
      res->mu = ps.mu;
      res->ms_schur += ps.ms_schur;
      res->ms_factor += ps.ms_factor;
      res->ms_other += ps.ms_other;
      // primal residual ||B(X) - a||_2
      Ipm* w = ipm_ws(c);
      call(polya_adjoint(ctx, st->X, w->tmpK, s), c);
      k_resid<<<kScalarBlocks, 256, 0, s>>>(c.K, w->tmpK, w->part);
      ++c.launches;
      CK(cudaGetLastError());
      CK(cudaMemcpyAsync(part.data(), w->part, kScalarBlocks * sizeof(double), cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      double r2 = 0.0;
      for (double v : part) r2 += v;
      res->pinf = std::sqrt(r2);
      if (!std::isfinite(res->gap) || !std::isfinite(res->pinf)) {
        res->status = POLYA_ENOTPD;
        return POLYA_OK;
      }
      if (res->gap <= opt->eps && res->pinf <= opt->tol) {   // stopping rule
        // every Z block positive definite (reading R10): the blockwise Cholesky of k_block_inv
        CK(cudaMemsetAsync(w->fail, 0, sizeof(int), s));
        const size_t smi = block_inv_smem(c.n);
        CK(cudaFuncSetAttribute(k_block_inv, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smi));
        k_block_inv<<<(unsigned)c.nb, 512, smi, s>>>((int)c.n, st->Z, w->W, w->fail);
        ++c.launches;
        CK(cudaGetLastError());
        int hfail = 0;
        CK(cudaMemcpyAsync(&hfail, w->fail, sizeof(int), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        res->converged = hfail ? 0 : 1;
        res->status = hfail ? POLYA_ENOTPD : POLYA_OK;
        return POLYA_OK;
      }
    }
  } catch (const IpmFail& f) {
    c.last_error = f.msg;
    return f.s;
  }
  return POLYA_OK;
}

extern "C" polya_status polya_verdict(polya_ctx* ctx, const double* y, int32_t npts, const double* pts_host,
                                      int32_t* nfail_out, void* stream) {
  if (!ctx || !y || npts < 0 || (npts > 0 && !pts_host) || !nfail_out) return POLYA_EINVAL;
  Ctx& c = ctx->c;
  const int64_t nextra = c.gen ? c.ncoef : c.nA;
  if ((c.n * c.n + c.L0 + nextra) * (int64_t)sizeof(double) > 227 * 1024) {
    c.last_error = "polya_verdict: n <= 168 (one n x n Cholesky matrix per point in shared memory)";
    return POLYA_EINVAL;
  }
  cudaStream_t s = (cudaStream_t)stream;
  *nfail_out = 0;
  if (npts == 0) return POLYA_OK;
  const int64_t per = (c.gen ? 5 : 3) * c.n * c.n;          // scratch doubles per point
  const int32_t chunk = (int32_t)std::max<int64_t>(1, std::min<int64_t>(npts, (int64_t)(1u << 28) / per));
  int32_t *dWp = nullptr, *dWa = nullptr, *dgen = nullptr;
  double *dpts = nullptr, *dscr = nullptr;
  int* dfail = nullptr;
  polya_status ret = POLYA_OK;
  try {
    CK(cudaMalloc(&dWp, c.Wp.size() * sizeof(int32_t)));
    CK(cudaMalloc(&dWa, c.Wa.size() * sizeof(int32_t)));
    CK(cudaMalloc(&dpts, (size_t)npts * c.l * sizeof(double)));
    CK(cudaMalloc(&dfail, sizeof(int)));
    CK(cudaMalloc(&dscr, (size_t)chunk * per * sizeof(double)));
    CK(cudaMemcpyAsync(dWp, c.Wp.data(), c.Wp.size() * sizeof(int32_t), cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(dWa, c.Wa.data(), c.Wa.size() * sizeof(int32_t), cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(dpts, pts_host, (size_t)npts * c.l * sizeof(double), cudaMemcpyHostToDevice, s));
    CK(cudaMemsetAsync(dfail, 0, sizeof(int), s));
    CK(launch_vmap(c, y, s));   // V_h(y) -> arena slots id_Vy + h
    const size_t sm = ((size_t)c.n * c.n + c.L0 + nextra) * sizeof(double);
    const int32_t* dexp = nullptr;
    const int32_t* dao = nullptr;
    const int nt = (int)c.gp_aoff.size();
    if (c.gen) {
      std::vector<int32_t> tab(c.coef_exp);   // [ncoef][l] exponents, then aoff[nt], boff[nt]
      tab.insert(tab.end(), c.gp_aoff.begin(), c.gp_aoff.end());
      tab.insert(tab.end(), c.gp_boff.begin(), c.gp_boff.end());
      CK(cudaMalloc(&dgen, tab.size() * sizeof(int32_t)));
      CK(cudaMemcpyAsync(dgen, tab.data(), tab.size() * sizeof(int32_t), cudaMemcpyHostToDevice, s));
      dexp = dgen;
      dao = dgen + c.coef_exp.size();
      CK(cudaFuncSetAttribute(k_grid_gen, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    } else {
      CK(cudaFuncSetAttribute(k_grid, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    }
    for (int32_t p0 = 0; p0 < npts; p0 += chunk) {   // points in chunks (bounded scratch)
      const int32_t cnt = std::min(chunk, npts - p0);
      const double* pp = dpts + (int64_t)p0 * c.l;
      if (c.gen)
        k_grid_gen<<<(unsigned)cnt, 256, sm, s>>>((int)c.n, (int)c.nbas, (int)c.l, (int)c.L0, nt, (int)c.ncoef,
                                                  (int)c.r_off, dWp, dexp, dao, dao + nt, c.d_coef, c.arena, c.mstride,
                                                  (int)c.np, c.id_Vy, pp, dscr, dfail);
      else
        k_grid<<<(unsigned)cnt, 256, sm, s>>>((int)c.n, (int)c.l, (int)c.L0, (int)c.nA, dWp, dWa, c.arena, c.mstride,
                                              (int)c.np, c.id_Vy, c.dA, pp, dscr, dfail);
      ++c.launches;
      CK(cudaGetLastError());
    }
    int h = 0;
    CK(cudaMemcpyAsync(&h, dfail, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    *nfail_out = h;
  } catch (const IpmFail& f) {
    c.last_error = f.msg;
    ret = f.s;
  }
  cudaFree(dWp);
  cudaFree(dWa);
  cudaFree(dgen);
  cudaFree(dpts);
  cudaFree(dscr);
  cudaFree(dfail);
  return ret;
}

extern "C" polya_status polya_set_factorization(polya_ctx* ctx, int mode) {
  if (!ctx || mode < 0 || mode > 2) return POLYA_EINVAL;
  ctx->c.fact_mode = mode;
  return POLYA_OK;
}
