// schur.cu -- kernel K4: assembly of the Schur complement matrix (SCM)
//     G_{(h,s),(h',t)} = sum_b tr(F_{(h,s)}^b W_b F_{(h',t)}^b X_b),   W = Z^{-1}
// (Eq. T2; the dominant decentralised cost, Case 1).
//
// Rank-structured expansion: for a pair (h, h') every block b contributes
// sum_k L_k[b1,c1] R_k[d1,a1], summed over the orientations (a1,b1) in or(s), (c1,d1) in or(t)
// of the basis elements s = {a,b}, t = {c,d}, with
//   Lyapunov m: (L,R) = (U_{h'}^T, V_h^T), (X, R_{h'h}), (Q_{hh'}, W), (U_h, V_{h'})
//   P-block  j: (L,R) = (beta_hj beta_h'j X, W)
// (U_h = H_h X, V_h = H_h W, Q_{hh'} = H_h X H_h'^T, R_{h'h} = H_h' W H_h^T; kernel K3).
// For fixed (h,h'), Raw[(x,y),(z,w)] = sum_k L_k[x,y] R_k[z,w] is a plain GEMM over k
// (M = N = n^2, inner dimension K_pair = 4 mu_hh' + nu_hh') and G is a fold of Raw in which
// every raw entry is added to exactly one G entry.
//
// Work item = (pair, row class {i<=j}, column class {k<=l}) of 8-index chunks.  A CTA of 4 warps
// computes the <= 4 raw 64x64 sub-blocks of the item (one per orientation) with FP64 DMMA
// (mma.sync m8n8k4 -> DMMA.8x8x4; sm_100a has no f64 tcgen05 kind), each warp a 4x4 grid of
// 8x8 MMA tiles.  Operands go global -> registers -> shared memory in a k-interleaved layout
// [x][y][slot(k)] so one LDS.128 feeds the fragments of two k-steps (8 LDS.128 per 32 DMMA);
// loads of stage s+1 are in flight while stage s computes.  Each orientation is folded into a
// 32 KB XOR-swizzled shared G-block (conflict-free for all four orientations), and the item's
// G entries are written with diagonal-ordered (contiguous-run) stores plus mirror stores.
// Persistent CTAs pull items from an atomic counter in pair-major order so co-running CTAs
// share a pair's operands in L2.  Every G entry is produced by one CTA in a fixed k order:
// deterministic, and FULL layouts are bitwise symmetric.
#include <algorithm>

#include "polya_internal.h"

namespace polya {
namespace {

constexpr int Q = kChunk;  // 8
constexpr int KB = 8;      // k terms per pipeline stage
constexpr int NT = 128;    // 4 warps
constexpr int KS = 68;     // doubles per staged 8x8 tile: 64 + 4 pad (conflict-free LDS.64 fragments)
constexpr int STAGE = 2 * KB * KS;  // doubles per stage: L[8 k][8 x][8 y] + R[8 k][8 z][8 w]
constexpr size_t kSmemBytes = (2 * STAGE + Q * Q * Q * Q) * sizeof(double);

struct SchurArgs {
  const double* arena;
  int64_t ms;
  unsigned ms32;   // np*np (< 2^32, checked at set-up): 32x32->64-bit address multiplies
  int np, n, ncls, npl;
  const int32_t* cls_a;
  const int32_t* cls_b;
  const int32_t* pair_h;
  const int32_t* pair_h2;
  const int64_t* pair_kbeg;
  const int64_t* pair_item;
  const int2* kdesc;
  int64_t item0, item1;
  unsigned long long* counter;
  double* G;
  int layout;
  int64_t K, Ntil;
};

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ int64_t svec_idx(int a, int b, int n) {
  const int o = b - a;
  if (o == 0) return a;
  return (int64_t)n + (int64_t)(o - 1) * n - (int64_t)(o - 1) * o / 2 + a;
}

// Shared G-block address of local (a,b,c,d): 16-double groups indexed by (a, b, c>>1), the low
// 4 bits (c&1, d) XOR-swizzled by a GF(2)-linear function of (a, b, c>>1), chosen by search
// so that the 32 lanes of every fold orientation hit distinct bank pairs.
// Every field is a bit field or an XOR, so the address splits into per-coordinate terms:
//   gs(a,b,c,d) = Ta(a) ^ Tb(b) ^ Tc(c) ^ d.
__device__ __forceinline__ int Ta(int a) {
  const int a0 = a & 1, a1 = (a >> 1) & 1, a2 = a >> 2;
  return (a << 9) ^ ((a0 ^ a1) | (a2 << 1) | ((a0 ^ a2) << 2) | ((a0 ^ a1 ^ a2) << 3));
}
__device__ __forceinline__ int Tb(int b) {
  const int b0 = b & 1, b1 = (b >> 1) & 1, b2 = b >> 2;
  return (b << 6) ^ ((b1 ^ b2) | ((b0 ^ b1 ^ b2) << 1) | (b2 << 2) | ((b0 ^ b1 ^ b2) << 3));
}
__device__ __forceinline__ int Tc(int c) {
  const int c1 = c >> 1, e0 = c1 & 1, e1 = c1 >> 1;
  return (c1 << 4) ^ ((c & 1) << 3) ^ (e1 | ((e0 ^ e1) << 1) | (e0 << 2));
}

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gmem_src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(gmem_src));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;\n" ::); }

__global__ void __launch_bounds__(NT, 4) k_schur(const SchurArgs p) {
  extern __shared__ __align__(16) double smem[];
  double* Gs = smem + 2 * STAGE;
  __shared__ unsigned char s_diag[64][2];  // (lc, ld) of local pairs ordered by (ld-lc, lc)
  __shared__ long long s_item;
  __shared__ int s_row[64], s_col[64];     // svec index of local (a,b) / (c,d) pairs, -1 if unused

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, t = lane & 3;
  if (tid < 64) {  // diagonal order: consecutive entries have consecutive svec indices
    int idx = 0;
    for (int dlt = -(Q - 1); dlt <= Q - 1; ++dlt)
      for (int lc = max(0, -dlt); lc <= min(Q - 1, Q - 1 - dlt); ++lc, ++idx)
        if (idx == tid) { s_diag[tid][0] = (unsigned char)lc; s_diag[tid][1] = (unsigned char)(lc + dlt); }
  }
  // cp.async tasks of this thread per stage: 16-byte chunk (row sr, column pair sc2) of the tiles
  // k = warp and k = warp + 4 of both operands
  const int sr = lane >> 2, sc2 = lane & 3;
  const int xw = 4 * (warp >> 1), zw = 4 * (warp & 1);  // warp's 4 x-tiles and 4 z-tiles

  for (;;) {
    if (tid == 0) s_item = (long long)atomicAdd(p.counter, 1ULL) + p.item0;
    __syncthreads();
    const int64_t item = s_item;
    __syncthreads();
    if (item >= p.item1) break;

    int pl = 0;
    {
      int lo = 0, hi = p.npl;
      while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (p.pair_item[mid] <= item) lo = mid; else hi = mid;
      }
      pl = lo;
    }
    const int h = p.pair_h[pl], h2 = p.pair_h2[pl];
    const int64_t rem = item - p.pair_item[pl];
    int sc, tc;
    if (h != h2) {
      sc = (int)(rem / p.ncls);
      tc = (int)(rem - (int64_t)sc * p.ncls);
    } else {
      int64_t r = rem;
      int s = 0;
      while (r >= p.ncls - s) { r -= p.ncls - s; ++s; }
      sc = s;
      tc = s + (int)r;
    }
    const int ci = p.cls_a[sc], cj = p.cls_b[sc], ck = p.cls_a[tc], cl = p.cls_b[tc];
    const bool dS = (ci == cj), dT = (ck == cl);
    const int64_t kb = p.pair_kbeg[pl];
    const int nstage = (int)((p.pair_kbeg[pl + 1] - kb) / KB);   // k-lists are padded to whole stages
    const int n = p.n, np = p.np;

    bool first = true;
    for (int o = 0; o < 4; ++o) {
      if ((o & 1) && dT) continue;
      if ((o & 2) && dS) continue;
      // Raw[(x,y),(z,w)], x in chunk cX, y in cY, z in cZ, w in cW; local G index (a,b,c,d) =
      //   o0: (w,x,y,z)  o1: (w,x,z,y)  o2: (x,w,y,z)  o3: (x,w,z,y)
      const int cX = (o & 2) ? ci : cj;
      const int cW = (o & 2) ? cj : ci;
      const int cY = (o & 1) ? cl : ck;
      const int cZ = (o & 1) ? ck : cl;
      const int nvx = min(Q, n - cX * Q), nvz = min(Q, n - cZ * Q);
      const int offL = (cX * Q + sr) * np + cY * Q + 2 * sc2;      // this thread's source offsets
      const int offR = (cZ * Q + sr) * np + cW * Q + 2 * sc2;
      const int dstT = sr * Q + 2 * sc2;                            // and target within a tile

      double acc[4][4][2];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
      // a warp whose x- or z-tiles all lie past a ragged chunk's end only multiplies zeros: skip
      const bool active = (xw < nvx) && (zw < nvz);

      // 2-stage cp.async pipeline; the descriptors (arena matrix ids of L_k, R_k) of the next
      // stage are fetched one stage ahead so no load waits on a dependent load
      int2 dc[2], dn[2];
      auto load_desc = [&](int s, int2* d) {
        if (s < nstage) {
          d[0] = __ldg(p.kdesc + kb + (int64_t)s * KB + warp);
          d[1] = __ldg(p.kdesc + kb + (int64_t)s * KB + warp + 4);
        }
      };
      auto issue = [&](int buf) {
        double* T = smem + buf * STAGE + dstT;
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int kk = warp + 4 * q;
          cp_async16(T + kk * KS, p.arena + (uint64_t)(unsigned)dc[q].x * p.ms32 + offL);
          cp_async16(T + KB * KS + kk * KS, p.arena + (uint64_t)(unsigned)dc[q].y * p.ms32 + offR);
        }
      };

      if (nstage > 0) {
        load_desc(0, dc);
        issue(0);
        cp_async_commit();
        load_desc(1, dc);
        const double* fA = smem + t * KS + xw * Q + g;   // fragment bases: A[y=g][k=t] of x-tile xw
        const double* fB = smem + KB * KS + t * KS + zw * Q + g;
        for (int s = 0; s < nstage; ++s) {
          const int boff = (s & 1) * STAGE;
          if (s + 1 < nstage) {
            issue((s & 1) ^ 1);      // stage s+1 (descriptors arrived during stage s-1)
            load_desc(s + 2, dn);
          }
          cp_async_commit();
          cp_async_wait1();          // this thread's copies of stage s have landed
          __syncthreads();           // ... and everybody else's
          if (active) {
#pragma unroll
            for (int k4 = 0; k4 < 2; ++k4) {
              double a[4], b[4];
#pragma unroll
              for (int i = 0; i < 4; ++i) a[i] = fA[boff + k4 * 4 * KS + i * Q];
#pragma unroll
              for (int j = 0; j < 4; ++j) b[j] = fB[boff + k4 * 4 * KS + j * Q];
#pragma unroll
              for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
            }
          }
          __syncthreads();           // buffer s&1 is refilled by the issue of iteration s+1
          dc[0] = dn[0]; dc[1] = dn[1];
        }
      }
      // fold: thread holds Raw(x = xw+i, y = g, z = zw+j, w = 2t+e) -> Gs[(a,b,c,d)(o)]
      {
        int bx[4], bz[4], be[2];
#pragma unroll
        for (int i = 0; i < 4; ++i) bx[i] = (o & 2) ? Ta(xw + i) : Tb(xw + i);
#pragma unroll
        for (int j = 0; j < 4; ++j) bz[j] = (o & 1) ? Tc(zw + j) : (zw + j);
#pragma unroll
        for (int e = 0; e < 2; ++e) be[e] = ((o & 2) ? Tb(2 * t + e) : Ta(2 * t + e)) ^ ((o & 1) ? g : Tc(g));
        if (first) {
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j)
#pragma unroll
              for (int e = 0; e < 2; ++e) Gs[be[e] ^ bx[i] ^ bz[j]] = acc[i][j][e];
        } else {
#pragma unroll
          for (int i = 0; i < 4; ++i) {  // 8 independent read-modify-writes at a time
            double old[4][2];
#pragma unroll
            for (int j = 0; j < 4; ++j)
#pragma unroll
              for (int e = 0; e < 2; ++e) old[j][e] = Gs[be[e] ^ bx[i] ^ bz[j]];
#pragma unroll
            for (int j = 0; j < 4; ++j)
#pragma unroll
              for (int e = 0; e < 2; ++e) Gs[be[e] ^ bx[i] ^ bz[j]] = old[j][e] + acc[i][j][e];
          }
        }
      }
      first = false;
      __syncthreads();
    }

    // ---- epilogue: fold diagonal classes and write G ----------------------------------------
    if (tid < 128) {  // svec tables of the item's local pairs
      const int q = tid & 63;
      const int l1 = q >> 3, l2 = q & 7;
      const int c1 = (tid < 64) ? ci : ck, c2 = (tid < 64) ? cj : cl;
      const bool dg = (tid < 64) ? dS : dT;
      const int a = c1 * Q + l1, b = c2 * Q + l2;
      const int v = (a < n && b < n && (!dg || l1 <= l2)) ? (int)svec_idx(a, b, n) : -1;
      if (tid < 64) s_row[q] = v; else s_col[q] = v;
    }
    __syncthreads();
    const bool diag_pair = (h == h2);
    const bool same_cls = diag_pair && (sc == tc);
    const int64_t rowbase = (int64_t)h * p.Ntil, colbase = (int64_t)h2 * p.Ntil;
    double* tile = p.G + (int64_t)pl * p.Ntil * p.Ntil;
    for (int pass = 0; pass < 2; ++pass) {
      // pass 0: direct entries, lanes along t (diagonal order); pass 1: mirror entries, lanes along s
      if (pass == 1 && !(p.layout == POLYA_G_FULL || diag_pair)) break;
      const int fa = s_diag[tid & 63][0], fb = s_diag[tid & 63][1];   // this thread's fixed pair
      const int fidx = pass == 0 ? s_col[fa * Q + fb] : s_row[fa * Q + fb];
      if (fidx < 0) continue;
      const int f_direct = pass == 0 ? (Tc(fa) ^ fb) : (Ta(fa) ^ Tb(fb));
      const int f_swap = pass == 0 ? (Tc(fb) ^ fa) : (Ta(fb) ^ Tb(fa));
      const bool fdiag = pass == 0 ? dT : dS;   // the fixed pair's class is diagonal
      const bool vdiag = pass == 0 ? dS : dT;   // the varying pair's class is diagonal
      for (int sl = tid >> 6; sl < 64; sl += NT / 64) {
        const int u1 = sl >> 3, u2 = sl & 7;
        const int vidx = pass == 0 ? s_row[sl] : s_col[sl];
        if (vidx < 0) continue;
        const int64_t s_ = pass == 0 ? vidx : fidx, t_ = pass == 0 ? fidx : vidx;
        if (same_cls && s_ > t_) continue;
        const int v_direct = pass == 0 ? (Ta(u1) ^ Tb(u2)) : (Tc(u1) ^ u2);
        const int v_swap = pass == 0 ? (Ta(u2) ^ Tb(u1)) : (Tc(u2) ^ u1);
        // canonical summation order (direct, s-swap, t-swap, both) in both passes, so that an
        // entry and its mirror image are bitwise equal
        const int s_d = pass == 0 ? v_direct : f_direct, s_s = pass == 0 ? v_swap : f_swap;
        const int t_d = pass == 0 ? f_direct : v_direct, t_s = pass == 0 ? f_swap : v_swap;
        const bool hs = pass == 0 ? (vdiag && u1 != u2) : (fdiag && fa != fb);
        const bool ht = pass == 0 ? (fdiag && fa != fb) : (vdiag && u1 != u2);
        double val = Gs[s_d ^ t_d];
        if (hs) val += Gs[s_s ^ t_d];
        if (ht) val += Gs[s_d ^ t_s];
        if (hs && ht) val += Gs[s_s ^ t_s];
        if (p.layout == POLYA_G_FULL) {
          if (pass == 0) p.G[(rowbase + s_) * p.K + colbase + t_] = val;
          else p.G[(colbase + t_) * p.K + rowbase + s_] = val;
        } else {
          if (pass == 0) tile[s_ * p.Ntil + t_] = val;
          else tile[t_ * p.Ntil + s_] = val;
        }
      }
    }
    // Gs / s_row / s_col are rewritten by the next item only after the syncs at the loop top
  }
}

}  // namespace

cudaError_t launch_schur(Ctx& c, double* G, int layout, cudaStream_t s) {
  if (c.item1 <= c.item0) return cudaSuccess;
  cudaError_t e = cudaMemsetAsync(c.st.counter, 0, sizeof(unsigned long long), s);
  if (e != cudaSuccess) return e;
  static bool attr_set = false;
  if (!attr_set) {
    e = cudaFuncSetAttribute(k_schur, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_schur, NT, kSmemBytes);
  per_sm = std::max(per_sm, 1);
  const int64_t want = std::min<int64_t>((int64_t)sms * per_sm, c.item1 - c.item0);
  SchurArgs a;
  a.arena = c.arena; a.ms = c.mstride; a.ms32 = (unsigned)c.mstride; a.np = (int)c.np; a.n = (int)c.n; a.ncls = (int)c.ncls;
  a.npl = (int)c.npairs_local;
  a.cls_a = c.st.cls_a; a.cls_b = c.st.cls_b; a.pair_h = c.st.pair_h; a.pair_h2 = c.st.pair_h2;
  a.pair_kbeg = c.st.pair_kbeg; a.pair_item = c.st.pair_item; a.kdesc = c.st.kdesc;
  a.item0 = c.item0; a.item1 = c.item1; a.counter = c.st.counter;
  a.G = G; a.layout = layout; a.K = c.K; a.Ntil = c.Ntil;
  k_schur<<<(unsigned)want, NT, kSmemBytes, s>>>(a);
  ++c.launches;
  return cudaGetLastError();
}

}  // namespace polya
