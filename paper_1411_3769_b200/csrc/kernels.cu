// kernels.cu -- set-up, operator and batched-GEMM kernels for sm_100a.
//
// K1 setup_H    : H_{h,gamma} = sum_lambda multinomial(d2; gamma-h-lambda) A_lambda (Eq. H)
// pad_copy      : caller block stack [nb][n][n] -> zero-padded np x np arena matrices
// K3 gemm       : batched C = sum_t alpha_t A_t op(B_t) on np x np arena matrices, FP64 DMMA (mma.sync
//                 m8n8k4 f64; tcgen05 has no f64 kind on sm_100a), used for the SCM precompute
//                 (U, V, Q, R), the forward map and the adjoint
// K8 vmap/apply : B^T(y) blocks (Eq. AT with Eq. 31)
// K9 adjoint    : B(X)_i = sum_b tr(F_i^b X_b), segmented reduction over blocks
#include <algorithm>

#include <cassert>

#include "polya_internal.h"

namespace polya {
namespace {

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// svec position of the basis element (a, b), a <= b, under reading R2 (diagonal-major).
__device__ __forceinline__ int64_t svec_idx(int a, int b, int n) {
  const int o = b - a;
  if (o == 0) return a;
  return (int64_t)n + (int64_t)(o - 1) * n - (int64_t)(o - 1) * o / 2 + a;
}

__global__ void k_setup_H(double* __restrict__ arena, int64_t ms, int np, int n, int nA,
                          const double* __restrict__ A, const double* __restrict__ Hw, int64_t id_H) {
  const int t = blockIdx.x;
  double* H = arena + (id_H + t) * ms;
  const double* w = Hw + (int64_t)t * nA;
  for (int e = threadIdx.x; e < np * np; e += blockDim.x) {
    const int i = e / np, j = e - i * np;
    double v = 0.0;
    if (i < n && j < n)
      for (int a = 0; a < nA; ++a) v += w[a] * A[((int64_t)a * n + i) * n + j];
    H[e] = v;
  }
}

// Generalised form (reading R18): dst = sum_q w_q coef[src_q] (trans: its transpose), zero-padded.
__global__ void k_wsum(double* __restrict__ arena, int64_t ms, int np, int n, const double* __restrict__ coef,
                       const WsumItem* __restrict__ items, const WsumTerm* __restrict__ terms) {
  const WsumItem it = items[blockIdx.x];
  double* D = arena + (int64_t)it.dst * ms;
  const int64_t nn = (int64_t)n * n;
  for (int e = threadIdx.x; e < np * np; e += blockDim.x) {
    const int i = e / np, j = e - i * np;
    double v = 0.0;
    if (i < n && j < n) {
      const int64_t off = it.trans ? (int64_t)j * n + i : (int64_t)i * n + j;
      for (int q = it.beg; q < it.end; ++q) v += terms[q].w * coef[terms[q].src * nn + off];
    }
    D[e] = v;
  }
}

__global__ void k_pad_copy(double* __restrict__ arena, int64_t ms, int np, int n, const double* __restrict__ src,
                           int64_t id0, int sym) {
  const int64_t b = blockIdx.x;
  double* dst = arena + (id0 + b) * ms;
  const double* s = src + b * n * n;
  for (int e = threadIdx.x; e < np * np; e += blockDim.x) {
    const int i = e / np, j = e - i * np;
    double v = 0.0;
    if (i < n && j < n) v = sym ? 0.5 * (s[i * n + j] + s[j * n + i]) : s[i * n + j];
    dst[e] = v;
  }
}

// dst_i = w_i * src_i on arena matrices (pre-scaled P-block copies beta_hj X_j, beta_hj W_j).
__global__ void k_scale_copy(double* __restrict__ arena, int64_t ms, const int32_t* __restrict__ dst,
                             const int32_t* __restrict__ src, const double* __restrict__ w) {
  const int e = blockIdx.x;
  const double2* s = reinterpret_cast<const double2*>(arena + (int64_t)src[e] * ms);
  double2* d = reinterpret_cast<double2*>(arena + (int64_t)dst[e] * ms);
  const double we = w[e];
  for (int64_t i = threadIdx.x; i < ms / 2; i += blockDim.x) {
    double2 v = s[i];
    d[i] = make_double2(we * v.x, we * v.y);
  }
}

// Batched GEMM on np x np arena matrices: C[c_id] = sum_terms alpha A[a_id] op(B[b_id]).  CTA = one
// 64x64 tile of one output matrix, 8 warps, each a 32x16 block = 4x2 DMMA m8n8 tiles (8x8 tiles that
// lie beyond np are skipped, warp-uniformly).  The K dimension of all terms is streamed in chunks
// of 16 through a 3-stage cp.async ring with one CTA barrier per chunk: A as [i][k] (row stride
// 20 doubles), B as [k][j] (stride 68) or, transposed, [j][k] (stride 20), so every fragment load
// of a half-warp hits 16 distinct bank pairs; k beyond np is zero-filled.
constexpr int GT = 64;               // output tile
constexpr int GK = 16;               // k per chunk
constexpr int GST = 3;               // ring stages
constexpr int AS = 20;               // [i][k] row stride (doubles), = 4 mod 16
constexpr int BSN = 68;              // [k][j] row stride, = 4 mod 16
constexpr int ABUF = GT * AS;        // 1280
constexpr int BBUF = GT * AS > GK * BSN ? GT * AS : GK * BSN;   // 1280 / 1088
constexpr size_t kGemmSmem = (size_t)GST * (ABUF + BBUF) * sizeof(double);
__device__ __forceinline__ void cp16z(void* dst, const void* src, bool valid) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src), "r"(valid ? 16 : 0));
}
__global__ void __launch_bounds__(256) k_gemm(double* __restrict__ arena, int64_t ms, int np,
                                              const GemmItem* __restrict__ items,
                                              const GemmTerm* __restrict__ terms, int tiles) {
  extern __shared__ __align__(16) double gsm[];
  double* As = gsm;                        // [GST][ABUF]
  double* Bs = gsm + GST * ABUF;           // [GST][BBUF]
  const GemmItem it = items[blockIdx.y];
  const int ti = blockIdx.x / tiles, tj = blockIdx.x - ti * tiles;
  const int i0 = ti * GT, j0 = tj * GT;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, t = lane & 3;
  const int wr = (warp >> 2) * 32, wc = (warp & 3) * 16;
  const int nkc = (np + GK - 1) / GK, total = (it.tend - it.tbeg) * nkc;
  auto issue = [&](int c, int buf) {
    const GemmTerm tm = terms[it.tbeg + c / nkc];
#ifdef POLYA_BOUNDS_CHECK
    assert(tm.a_id >= 0 && tm.b_id >= 0 && it.c_id >= 0 && (int64_t)tm.a_id * ms >= 0);
#endif
    const int k0 = (c % nkc) * GK;
    const double* A = arena + (int64_t)tm.a_id * ms;
    const double* B = arena + (int64_t)tm.b_id * ms;
    double* as = As + buf * ABUF;
    double* bs = Bs + buf * BBUF;
#pragma unroll
    for (int r = 0; r < 2; ++r) {   // A rows i0..i0+63, columns k0..k0+15: two 16-byte copies per thread
      const int q = tid + r * 256, i = q >> 3, kc = (q & 7) * 2;
      const bool v = i0 + i < np && k0 + kc < np;
      cp16z(&as[i * AS + kc], v ? A + (int64_t)(i0 + i) * np + k0 + kc : A, v);
    }
    if (!tm.transB) {  // B rows k0..k0+15, columns j0..j0+63
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int q = tid + r * 256, k = q >> 5, jc = (q & 31) * 2;
        const bool v = k0 + k < np && j0 + jc < np;
        cp16z(&bs[k * BSN + jc], v ? B + (int64_t)(k0 + k) * np + j0 + jc : B, v);
      }
    } else {           // op(B)[k][j] = B[j][k]: rows j0..j0+63 of B, columns k0..k0+15
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int q = tid + r * 256, j = q >> 3, kc = (q & 7) * 2;
        const bool v = j0 + j < np && k0 + kc < np;
        cp16z(&bs[j * AS + kc], v ? B + (int64_t)(j0 + j) * np + k0 + kc : B, v);
      }
    }
  };
  // warp-uniform validity of the warp's 8x8 tiles (rows / columns beyond np are never formed)
  bool mv[4], nv[2];
#pragma unroll
  for (int mi = 0; mi < 4; ++mi) mv[mi] = i0 + wr + mi * 8 < np;
#pragma unroll
  for (int nj = 0; nj < 2; ++nj) nv[nj] = j0 + wc + nj * 8 < np;
  double acc[4][2][2] = {};
#pragma unroll
  for (int p = 0; p < GST - 1; ++p) {
    if (p < total) issue(p, p);
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  }
  for (int c = 0; c < total; ++c) {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(GST - 2) : "memory");
    __syncthreads();   // chunk c landed for every thread; the buffer of chunk c-1 is free
    if (c + GST - 1 < total) issue(c + GST - 1, (c + GST - 1) % GST);
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    const int buf = c % GST;
    const double* as = As + buf * ABUF;
    const double* bs = Bs + buf * BBUF;
    const GemmTerm tm = terms[it.tbeg + c / nkc];
#pragma unroll
    for (int ks = 0; ks < GK / 4; ++ks) {
      double a[4], b[2];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) a[mi] = as[(wr + mi * 8 + g) * AS + ks * 4 + t] * tm.alpha;
#pragma unroll
      for (int nj = 0; nj < 2; ++nj)
        b[nj] = tm.transB ? bs[(wc + nj * 8 + g) * AS + ks * 4 + t] : bs[(ks * 4 + t) * BSN + wc + nj * 8 + g];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int nj = 0; nj < 2; ++nj)
          if (mv[mi] && nv[nj]) dmma(acc[mi][nj][0], acc[mi][nj][1], a[mi], b[nj]);
    }
  }
  double* C = arena + (int64_t)it.c_id * ms;
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int nj = 0; nj < 2; ++nj) {
      const int i = i0 + wr + mi * 8 + g, j = j0 + wc + nj * 8 + 2 * t;
      if (i < np && j < np) *reinterpret_cast<double2*>(C + (int64_t)i * np + j) = make_double2(acc[mi][nj][0], acc[mi][nj][1]);
    }
  if (it.ct_id >= 0) {   // the transpose as well (8 lanes of a row group store 64 contiguous bytes)
    double* Ct = arena + (int64_t)it.ct_id * ms;
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int nj = 0; nj < 2; ++nj) {
        const int i = i0 + wr + mi * 8 + g, j = j0 + wc + nj * 8 + 2 * t;
        if (i < np && j < np) {
          Ct[(int64_t)j * np + i] = acc[mi][nj][0];
          Ct[(int64_t)(j + 1) * np + i] = acc[mi][nj][1];
        }
      }
  }
}

// K3b: row-gathered GEMM for the SCM precompute (standard form, np <= 128).  U_t = H_t X_m for all t of
// one block m share X_m, and Q_{hh'} = U_h H_{h'}^T for all h paired with h' (one m) share H_{h'}: a group
// stacks the rows of its left operands (np rows each) and a CTA computes 64 stacked rows x all np columns
// (8 warps: 4 x 16 rows, 2 column halves of <= 8 8x8 tiles; 32 accumulators per thread), so the output
// tile is never ragged in the row direction except at a group's end and the column split is within one
// tile of even (np = 104: 7 + 6 tiles) -- vs 64x64 tiles of one np x np output, where np = 104 leaves
// 34 % of the warp tiles beyond np.  K streamed in chunks of 16 through a 3-stage cp.async ring, the
// conflict-free layouts of k_gemm ([i][k] stride 20; [k][j] stride 132 or, transposed, [j][k] stride 20).
constexpr int RT = 64;                  // stacked rows per CTA
constexpr int RBN = 132;                // [k][j] row stride (= 4 mod 16), np <= 128
constexpr int RABUF = RT * AS;          // 1280
constexpr int RBBUF = 128 * AS > GK * RBN ? 128 * AS : GK * RBN;   // 2560 / 2112
constexpr size_t kRgSmem = (size_t)GST * (RABUF + RBBUF) * sizeof(double);   // 92,160 bytes
template <bool TRANS>
__global__ void __launch_bounds__(256, 2) k_rgemm(double* __restrict__ arena, int64_t ms, int np,
                                                  const RgGroup* __restrict__ groups, const RgEnt* __restrict__ ents,
                                                  const RgTile* __restrict__ tiles) {
  extern __shared__ __align__(16) double gsm[];
  double* As = gsm;
  double* Bs = gsm + GST * RABUF;
  const RgTile tl = tiles[blockIdx.x];
  const RgGroup gr = groups[tl.group];
  const int rows = (gr.eend - gr.ebeg) * np;   // stacked rows of the group
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, t = lane & 3;
  const int wm = warp >> 1, wn = warp & 1;
  const int nt8 = np >> 3, nh = (nt8 + 1) >> 1;
  const int jc0 = wn * nh, ncw = wn ? nt8 - nh : nh;   // the warp's column tiles [jc0, jc0 + ncw)
  const double* B = arena + (int64_t)gr.b_id * ms;
  // the two stacked A rows this thread copies (fixed over the K loop)
  const double* arow[2];
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int R = tl.r0 + ((tid + r * 256) >> 3);
    arow[r] = nullptr;
    if (R < rows) {
      const int e = R / np;
      arow[r] = arena + (int64_t)ents[gr.ebeg + e].a_id * ms + (int64_t)(R - e * np) * np;
    }
  }
  const int nkc = (np + GK - 1) / GK;
  auto issue = [&](int c, int buf) {
    const int k0 = c * GK;
    double* as = As + buf * RABUF;
    double* bs = Bs + buf * RBBUF;
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int q = tid + r * 256, i = q >> 3, kc = (q & 7) * 2;
      const bool v = arow[r] != nullptr && k0 + kc < np;
      cp16z(&as[i * AS + kc], v ? arow[r] + k0 + kc : B, v);
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int q = tid + r * 256;
      if (!TRANS) {   // B rows k0..k0+15, columns 0..np-1
        const int k = q >> 6, jc = (q & 63) * 2;
        const bool v = k0 + k < np && jc < np;
        cp16z(&bs[k * RBN + jc], v ? B + (int64_t)(k0 + k) * np + jc : B, v);
      } else {        // op(B)[k][j] = B[j][k]: rows j of B, columns k0..k0+15
        const int j = q >> 3, kc = (q & 7) * 2;
        const bool v = j < np && k0 + kc < np;
        cp16z(&bs[j * AS + kc], v ? B + (int64_t)j * np + k0 + kc : B, v);
      }
    }
  };
  double acc[2][8][2] = {};
  bool mv[2];   // warp-uniform: the 8-row tile holds stacked rows of the group (not the padding of its last tile)
#pragma unroll
  for (int mi = 0; mi < 2; ++mi) mv[mi] = tl.r0 + wm * 16 + mi * 8 < rows;
#pragma unroll
  for (int p = 0; p < GST - 1; ++p) {
    if (p < nkc) issue(p, p);
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  }
  for (int c = 0; c < nkc; ++c) {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(GST - 2) : "memory");
    __syncthreads();   // chunk c landed for every thread; the buffer of chunk c-1 is free
    if (c + GST - 1 < nkc) issue(c + GST - 1, (c + GST - 1) % GST);
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    const double* as = As + (c % GST) * RABUF;
    const double* bs = Bs + (c % GST) * RBBUF;
#pragma unroll
    for (int ks = 0; ks < GK / 4; ++ks) {
      if (c * GK + ks * 4 >= np) break;   // np is a multiple of 8: the last chunk may hold 2 k-steps only
      double a[2], b[8];
#pragma unroll
      for (int mi = 0; mi < 2; ++mi) a[mi] = as[(wm * 16 + mi * 8 + g) * AS + ks * 4 + t];
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (j < ncw) {
          const int col = (jc0 + j) * 8 + g;
          b[j] = TRANS ? bs[col * AS + ks * 4 + t] : bs[(ks * 4 + t) * RBN + col];
        }
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (j < ncw) {
#pragma unroll
          for (int mi = 0; mi < 2; ++mi)
            if (mv[mi]) dmma(acc[mi][j][0], acc[mi][j][1], a[mi], b[j]);
        }
    }
  }
#pragma unroll
  for (int mi = 0; mi < 2; ++mi) {
    const int R = tl.r0 + wm * 16 + mi * 8 + g;
    if (R >= rows) continue;
    const int e = R / np, row = R - e * np;
    const RgEnt en = ents[gr.ebeg + e];
    double* C = arena + (int64_t)en.c_id * ms;
    double* Ct = en.ct_id >= 0 ? arena + (int64_t)en.ct_id * ms : nullptr;
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (j < ncw) {
        const int col = (jc0 + j) * 8 + 2 * t;
        *reinterpret_cast<double2*>(C + (int64_t)row * np + col) = make_double2(acc[mi][j][0], acc[mi][j][1]);
        if (Ct) {
          Ct[(int64_t)col * np + row] = acc[mi][j][0];
          Ct[(int64_t)(col + 1) * np + row] = acc[mi][j][1];
        }
      }
  }
}

// V_h(y) (Eq. 30) for every h into the arena (n = order of P; zero beyond it, reading R19).
__global__ void k_vmap(double* __restrict__ arena, int64_t ms, int np, int n, int64_t Ntil,
                       const double* __restrict__ y, int64_t id_Vy) {
  const int h = blockIdx.x;
  double* V = arena + (id_Vy + h) * ms;
  const double* yh = y + (int64_t)h * Ntil;
  for (int e = threadIdx.x; e < np * np; e += blockDim.x) {
    const int i = e / np, j = e - i * np;
    double v = 0.0;
    if (i < n && j < n) v = yh[svec_idx(min(i, j), max(i, j), n)];
    V[e] = v;
  }
}

// B^T(y) blocks: P-block j: sum_h beta_{h,j} V_h(y); Lyapunov m: -(S_m + S_m^T), S_m = sum_h V_h H_{h,m}.
// (n = block order, nbas = order of P: a P-block's LMI is its top-left nbas x nbas corner, R19)
__global__ void k_apply_out(const double* __restrict__ arena, int64_t ms, int np, int n, int nbas, int64_t Ntil,
                            int64_t L, const double* __restrict__ y, const int32_t* __restrict__ bP_beg,
                            const int32_t* __restrict__ bP_h, const double* __restrict__ bP_w, int64_t id_S,
                            double* __restrict__ out) {
  const int64_t b = blockIdx.x;
  double* o = out + b * n * n;
  if (b < L) {
    const int e0 = bP_beg[b], e1 = bP_beg[b + 1];
    for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
      const int i = e / n, j = e - i * n;
      double v = 0.0;
      if (i < nbas && j < nbas) {
        const int64_t k = svec_idx(min(i, j), max(i, j), nbas);
        for (int q = e0; q < e1; ++q) v += bP_w[q] * y[(int64_t)bP_h[q] * Ntil + k];
      }
      o[e] = v;
    }
  } else {
    const double* S = arena + (id_S + (b - L)) * ms;
    for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
      const int i = e / n, j = e - i * n;
      o[e] = -(S[i * np + j] + S[j * np + i]);
    }
  }
}

// y_(h,k) = sum_{j: beta_hj != 0} beta_hj [Xs_j]_k - 2 sum_{m: H_hm != 0} [H_hm Xs_m]_k,
// [M]_k = M_aa (k diagonal) or M_ab + M_ba, Xs = sym(X) (polya_adjoint), T_t = H_t Xs_m in the arena.
__global__ void k_adjoint_reduce(const double* __restrict__ arena, int64_t ms, int np, int n, int64_t Ntil,
                                 const int32_t* __restrict__ hP_beg, const int32_t* __restrict__ hP_j,
                                 const double* __restrict__ hP_w, const int32_t* __restrict__ hL_beg,
                                 const int32_t* __restrict__ hL_t, int64_t id_Xt, int64_t id_T,
                                 double* __restrict__ y) {
  const int h = blockIdx.y;
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= Ntil) return;
  // invert svec_idx: diagonal first, then offsets o = 1.. with n - o entries each
  int a, b;
  if (k < n) { a = b = (int)k; }
  else {
    int64_t r = k - n;
    int o = 1;
    while (r >= n - o) { r -= n - o; ++o; }
    a = (int)r;
    b = a + o;
  }
  const int64_t ab = (int64_t)a * np + b, ba = (int64_t)b * np + a;
  double v = 0.0;
  for (int q = hP_beg[h]; q < hP_beg[h + 1]; ++q) {
    const double* X = arena + (id_Xt + hP_j[q]) * ms;
    v += hP_w[q] * (a == b ? X[ab] : X[ab] + X[ba]);
  }
  for (int q = hL_beg[h]; q < hL_beg[h + 1]; ++q) {
    const double* T = arena + (id_T + hL_t[q]) * ms;
    v -= 2.0 * (a == b ? T[ab] : T[ab] + T[ba]);
  }
  y[(int64_t)h * Ntil + k] = v;
}

}  // namespace

cudaError_t launch_setup_H(Ctx& c, cudaStream_t s) {
  const int64_t nnzH = (int64_t)c.Hh.size();
  if (nnzH == 0) return cudaSuccess;
  k_setup_H<<<(unsigned)nnzH, 256, 0, s>>>(c.arena, c.mstride, (int)c.np, (int)c.n, (int)c.nA, c.dA, c.dHw, c.id_H);
  ++c.launches;
  return cudaGetLastError();
}

cudaError_t launch_wsum(Ctx& c, cudaStream_t s) {
  if (c.n_ws == 0) return cudaSuccess;
  k_wsum<<<(unsigned)c.n_ws, 256, 0, s>>>(c.arena, c.mstride, (int)c.np, (int)c.n, c.d_coef, c.d_ws_items, c.d_ws_terms);
  ++c.launches;
  return cudaGetLastError();
}

cudaError_t launch_pad_copy(Ctx& c, const double* src, int64_t id0, int64_t count, int sym, cudaStream_t s) {
  if (count == 0) return cudaSuccess;
  k_pad_copy<<<(unsigned)count, 256, 0, s>>>(c.arena, c.mstride, (int)c.np, (int)c.n, src, id0, sym);
  ++c.launches;
  return cudaGetLastError();
}

cudaError_t launch_scale_copy(Ctx& c, cudaStream_t s) {
  if (c.n_sc == 0) return cudaSuccess;
  k_scale_copy<<<(unsigned)c.n_sc, 256, 0, s>>>(c.arena, c.mstride, c.d_sc_dst, c.d_sc_src, c.d_sc_w);
  ++c.launches;
  return cudaGetLastError();
}

cudaError_t launch_gemm(Ctx& c, const GemmItem* items, const GemmTerm* terms, int64_t nitems, cudaStream_t s) {
  if (nitems == 0) return cudaSuccess;
  const int tiles = (int)((c.np + GT - 1) / GT);
  // per call (cheap): the attribute is per device, and a process may drive contexts on several
  cudaError_t e = cudaFuncSetAttribute(k_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kGemmSmem);
  if (e != cudaSuccess) return e;
  for (int64_t off = 0; off < nitems; off += 65535) {
    const int64_t cnt = std::min<int64_t>(65535, nitems - off);
    dim3 grid((unsigned)(tiles * tiles), (unsigned)cnt);
    k_gemm<<<grid, 256, kGemmSmem, s>>>(c.arena, c.mstride, (int)c.np, items + off, terms, tiles);
    ++c.launches;
  }
  return cudaGetLastError();
}

cudaError_t launch_rgemm(Ctx& c, int phase, cudaStream_t s) {
  const int64_t nt = c.n_rg_tile[phase];
  if (nt == 0) return cudaSuccess;
  // transB is uniform per launch: phases 0 (U, V) and 2 (T) multiply by X, W; phase 1 (Q, R) by H^T
  const bool trans = phase == 1;
  cudaError_t e = cudaFuncSetAttribute(trans ? k_rgemm<true> : k_rgemm<false>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kRgSmem);
  if (e != cudaSuccess) return e;
  if (trans)
    k_rgemm<true><<<(unsigned)nt, 256, kRgSmem, s>>>(c.arena, c.mstride, (int)c.np, c.d_rg_grp[phase], c.d_rg_ent[phase],
                                                      c.d_rg_tile[phase]);
  else
    k_rgemm<false><<<(unsigned)nt, 256, kRgSmem, s>>>(c.arena, c.mstride, (int)c.np, c.d_rg_grp[phase], c.d_rg_ent[phase],
                                                       c.d_rg_tile[phase]);
  ++c.launches;
  return cudaGetLastError();
}

cudaError_t launch_vmap(Ctx& c, const double* y, cudaStream_t s) {
  k_vmap<<<(unsigned)c.L0, 256, 0, s>>>(c.arena, c.mstride, (int)c.np, (int)c.nbas, c.Ntil, y, c.id_Vy);
  ++c.launches;
  return cudaGetLastError();
}

cudaError_t launch_apply_out(Ctx& c, const double* y, double* out, cudaStream_t s) {
  k_apply_out<<<(unsigned)c.nb, 256, 0, s>>>(c.arena, c.mstride, (int)c.np, (int)c.n, (int)c.nbas, c.Ntil, c.L, y, c.d_bP_beg,
                                              c.d_bP_h, c.d_bP_w, c.id_S, out);
  ++c.launches;
  return cudaGetLastError();
}

cudaError_t launch_adjoint_reduce(Ctx& c, double* y, cudaStream_t s) {
  dim3 grid((unsigned)((c.Ntil + 127) / 128), (unsigned)c.L0);
  k_adjoint_reduce<<<grid, 128, 0, s>>>(c.arena, c.mstride, (int)c.np, (int)c.nbas, c.Ntil, c.d_hP_beg, c.d_hP_j,
                                         c.d_hP_w, c.d_hL_beg, c.d_hL_t, c.id_Xt, c.id_T, y);
  ++c.launches;
  return cudaGetLastError();
}

// ---- the fused P2P combine of the block-sharded Schur complement (combine.cpp) ------------------
namespace {
__global__ void k_p2p_signal(int* const* flags, int n, int epoch) {
  const int r = threadIdx.x;
  if (r < n) {
    __threadfence_system();
    asm volatile("st.release.sys.global.b32 [%0], %1;\n" ::"l"(flags[r]), "r"(epoch) : "memory");
  }
}
// Spins until every flag reaches the epoch; a peer that never signals (it died, or a caller skipped a
// phase) ends in a trap after kP2pTimeoutNs instead of a hang: the launch then fails with a CUDA error.
constexpr unsigned long long kP2pTimeoutNs = 60ull * 1000000000ull;
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__global__ void k_p2p_wait(const int* flags, int n, int epoch) {
  const unsigned long long t0 = globaltimer();
  for (int r = 0; r < n; ++r)
    for (;;) {
      int v;
      asm volatile("ld.acquire.sys.global.b32 %0, [%1];\n" : "=r"(v) : "l"(flags + r) : "memory");
      if (v >= epoch) break;
      if (globaltimer() - t0 > kP2pTimeoutNs) __trap();
      __nanosleep(256);
    }
}
__global__ void k_p2p_sum(const double* __restrict__ slots, int n, int64_t count, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    double v = __ldcv(slots + i);   // written by peers: bypass L1
    for (int r = 1; r < n; ++r) v += __ldcv(slots + r * count + i);   // rank order
    out[i] = v;
  }
}
}  // namespace

cudaError_t launch_p2p_signal(int* const* flag_ptrs, int n, int epoch, cudaStream_t s) {
  k_p2p_signal<<<1, 32 * ((n + 31) / 32), 0, s>>>(flag_ptrs, n, epoch);
  return cudaGetLastError();
}
cudaError_t launch_p2p_wait(const int* flags, int n, int epoch, cudaStream_t s) {
  k_p2p_wait<<<1, 1, 0, s>>>(flags, n, epoch);
  return cudaGetLastError();
}
cudaError_t launch_p2p_sum(const double* slots, int n, int64_t count, double* out, cudaStream_t s) {
  const int64_t blocks = std::min<int64_t>((count + 255) / 256, 148 * 16);
  k_p2p_sum<<<(unsigned)std::max<int64_t>(blocks, 1), 256, 0, s>>>(slots, n, count, out);
  return cudaGetLastError();
}

}  // namespace polya
