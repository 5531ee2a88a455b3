// schur.cu -- kernel K4: assembly of the Schur complement matrix (SCM)
//     G_{(h,s),(h',t)} = sum_b tr(F_{(h,s)}^b W_b F_{(h',t)}^b X_b),   W = Z^{-1}
// (Eq. T2; the dominant decentralised cost, Case 1).
//
// Rank-structured expansion: for a pair (h, h') every block b
// contributes terms  sum_{k} L_k[b1,c1] R_k[d1,a1]  summed over the orientations
// (a1,b1) in or(s), (c1,d1) in or(t) of the basis elements s = {a,b}, t = {c,d}, with
//   Lyapunov m: (L,R) = (U_{h'}^T, V_h^T), (X, R_{h'h}), (Q_{hh'}, W), (U_h, V_{h'})
//   P-block  j: (L,R) = (beta_hj beta_h'j X, W)
// (U_h = H_h X, V_h = H_h W, Q_{hh'} = H_h X H_h'^T, R_{h'h} = H_h' W H_h^T; kernel K3).
// So for fixed (h,h'), Raw[(x,y),(z,w)] = sum_k L_k[x,y] R_k[z,w] is a plain GEMM over k
// (M = N = n^2, inner dimension K_pair = 4 mu_hh' + nu_hh') and G is a "fold" of Raw in which
// every Raw entry is added to exactly one G entry.
//
// Work item = (pair, row class {i<=j}, column class {k<=l}) of index chunks of size 8.  The CTA
// computes the <= 4 raw sub-blocks (64 x 64 each, one per orientation) with FP64 DMMA
// (mma.sync m8n8k4; the sm_100a FP64 tensor path -- tcgen05 has no f64 kind), folds them in
// shared memory and writes the G entries (and their mirror images).  Persistent CTAs pull work
// items from an atomic counter; items are ordered pair-major so CTAs running together share the
// pair's operands in L2.  Each G entry is produced by exactly one CTA in a fixed k order:
// the result is deterministic and FULL layouts are bitwise symmetric.
#include <algorithm>

#include "polya_internal.h"

namespace polya {
namespace {

constexpr int Q = kChunk;  // 8
constexpr int KB = 8;      // k terms per pipeline stage
constexpr int TS = 72;     // doubles per staged 8x8 tile (+8 pad: conflict-free fragment loads)
constexpr int NT = 256;    // 8 warps; warp w owns raw row-tile x = w
constexpr size_t kSmemBytes = (4 * KB * TS + Q * Q * Q * Q) * sizeof(double);

struct SchurArgs {
  const double* arena;
  int64_t ms;
  int np, n, ncls, npl;
  const int32_t* cls_a;
  const int32_t* cls_b;
  const int32_t* pair_h;
  const int32_t* pair_h2;
  const int64_t* pair_kbeg;
  const int64_t* pair_item;
  const int32_t* kL;
  const int32_t* kR;
  const int32_t* kf;
  const double* ks;
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

__global__ void __launch_bounds__(NT, 2) k_schur(const SchurArgs p) {
  extern __shared__ __align__(16) double smem[];
  double (*Ls)[KB * TS] = reinterpret_cast<double (*)[KB * TS]>(smem);
  double (*Rs)[KB * TS] = reinterpret_cast<double (*)[KB * TS]>(smem + 2 * KB * TS);
  double* Gs = smem + 4 * KB * TS;
  __shared__ unsigned char s_diag[64][2];  // (lc, ld) of local column pairs ordered by (ld-lc, lc)
  __shared__ long long s_item;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, t = lane & 3;
  if (tid < 64) {  // diagonal order: consecutive entries have consecutive svec indices
    int idx = 0;
    for (int dlt = -(Q - 1); dlt <= Q - 1; ++dlt)
      for (int lc = max(0, -dlt); lc <= min(Q - 1, Q - 1 - dlt); ++lc, ++idx)
        if (idx == tid) { s_diag[tid][0] = (unsigned char)lc; s_diag[tid][1] = (unsigned char)(lc + dlt); }
  }

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
    const int64_t kb = p.pair_kbeg[pl], ke = p.pair_kbeg[pl + 1];
    const int nstage = (int)((ke - kb + KB - 1) / KB);

    bool first = true;
    for (int o = 0; o < 4; ++o) {
      if ((o & 1) && dT) continue;
      if ((o & 2) && dS) continue;
      // Raw[(x,y),(z,w)], x in cX, y in cY, z in cZ, w in cW; local G index (a,b,c,d) =
      //   o0: (w,x,y,z)  o1: (w,x,z,y)  o2: (x,w,y,z)  o3: (x,w,z,y)
      const int cX = (o & 2) ? ci : cj;
      const int cW = (o & 2) ? cj : ci;
      const int cY = (o & 1) ? cl : ck;
      const int cZ = (o & 1) ? ck : cl;

      double acc[8][2];
#pragma unroll
      for (int d = 0; d < 8; ++d) acc[d][0] = acc[d][1] = 0.0;

      // staging: thread -> 2 x 16 B of the 16 tiles (8 L + 8 R) of a stage
      double2 v[2];
      int trf[2];
      auto load = [&](int s) {
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int pidx = tid + NT * u, tile = pidx >> 5, kk = tile & 7, isR = tile >> 3;
          const int within = pidx & 31, rr = within >> 2, cc = (within & 3) * 2;
          const int64_t k = kb + (int64_t)s * KB + kk;
          v[u] = make_double2(0.0, 0.0);
          trf[u] = 0;
          if (k < ke) {
            const int id = isR ? p.kR[k] : p.kL[k];
            const int tr = (p.kf[k] >> isR) & 1;
            const int rch = isR ? cZ : cX, cch = isR ? cW : cY;
            const int r0 = (tr ? cch : rch) * Q, c0 = (tr ? rch : cch) * Q;
            v[u] = __ldg(reinterpret_cast<const double2*>(p.arena + (int64_t)id * p.ms + (int64_t)(r0 + rr) * p.np + c0 + cc));
            if (!isR) {
              const double sc_ = __ldg(p.ks + k);
              v[u].x *= sc_;
              v[u].y *= sc_;
            }
            trf[u] = tr;
          }
        }
      };
      auto store = [&](int buf) {
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int pidx = tid + NT * u, tile = pidx >> 5, kk = tile & 7, isR = tile >> 3;
          const int within = pidx & 31, rr = within >> 2, cc = (within & 3) * 2;
          double* T = (isR ? Rs[buf] : Ls[buf]) + kk * TS;
          if (!trf[u]) {
            *reinterpret_cast<double2*>(T + rr * Q + cc) = v[u];
          } else {
            T[cc * Q + rr] = v[u].x;
            T[(cc + 1) * Q + rr] = v[u].y;
          }
        }
      };

      if (nstage > 0) {
        load(0);
        store(0);
        __syncthreads();
        for (int s = 0; s < nstage; ++s) {
          const int buf = s & 1;
          if (s + 1 < nstage) load(s + 1);
          const double* Lb = Ls[buf];
          const double* Rb = Rs[buf];
#pragma unroll
          for (int k4 = 0; k4 < KB / 4; ++k4) {
            const int kk = k4 * 4 + t;
            const double a = Lb[kk * TS + warp * Q + g];
#pragma unroll
            for (int d = 0; d < 8; ++d) {
              const double b = Rb[kk * TS + d * Q + g];
              dmma(acc[d][0], acc[d][1], a, b);
            }
          }
          if (s + 1 < nstage) store(buf ^ 1);
          __syncthreads();
        }
      }
      // fold this orientation into Gs: thread holds Raw(x=warp, y=g, z=d, w=2t+e)
#pragma unroll
      for (int d = 0; d < 8; ++d)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int x = warp, y = g, z = d, w = 2 * t + e;
          int la, lb, lc, ld;
          if (o & 2) { la = x; lb = w; } else { la = w; lb = x; }
          if (o & 1) { lc = z; ld = y; } else { lc = y; ld = z; }
          const int gi = ((la * Q + lb) * Q + lc) * Q + ld;
          if (first) Gs[gi] = acc[d][e]; else Gs[gi] += acc[d][e];
        }
      first = false;
      __syncthreads();
    }

    // ---- epilogue: fold diagonal classes and write G ----------------------------------------
    const int n = p.n;
    const bool diag_pair = (h == h2);
    const bool same_cls = diag_pair && (sc == tc);
    const int64_t rowbase = (int64_t)h * p.Ntil, colbase = (int64_t)h2 * p.Ntil;
    double* tile = p.G + (int64_t)pl * p.Ntil * p.Ntil;
    for (int pass = 0; pass < 2; ++pass) {
      // pass 0: direct entries, consecutive threads along t; pass 1: mirror entries along s
      if (pass == 1 && !(p.layout == POLYA_G_FULL || diag_pair)) break;
      for (int e = tid; e < 64 * 64; e += NT) {
        int la, lb, lc, ld;
        if (pass == 0) {
          la = (e >> 6) >> 3; lb = (e >> 6) & 7;
          lc = s_diag[e & 63][0]; ld = s_diag[e & 63][1];
        } else {
          lc = (e >> 6) >> 3; ld = (e >> 6) & 7;
          la = s_diag[e & 63][0]; lb = s_diag[e & 63][1];
        }
        if (dS && la > lb) continue;
        if (dT && lc > ld) continue;
        const int a = ci * Q + la, b = cj * Q + lb, c = ck * Q + lc, d = cl * Q + ld;
        if (a >= n || b >= n || c >= n || d >= n) continue;
        const int64_t s_ = svec_idx(a, b, n), t_ = svec_idx(c, d, n);
        if (same_cls && s_ > t_) continue;
        double v = Gs[((la * Q + lb) * Q + lc) * Q + ld];
        if (dS && la != lb) v += Gs[((lb * Q + la) * Q + lc) * Q + ld];
        if (dT && lc != ld) v += Gs[((la * Q + lb) * Q + ld) * Q + lc];
        if (dS && dT && la != lb && lc != ld) v += Gs[((lb * Q + la) * Q + ld) * Q + lc];
        if (p.layout == POLYA_G_FULL) {
          if (pass == 0) p.G[(rowbase + s_) * p.K + colbase + t_] = v;
          else p.G[(colbase + t_) * p.K + rowbase + s_] = v;
        } else {
          if (pass == 0) tile[s_ * p.Ntil + t_] = v;
          else tile[t_ * p.Ntil + s_] = v;
        }
      }
    }
    // Gs is rewritten by the next item only after the syncs at the top of the loop
  }
}

}  // namespace

cudaError_t launch_schur(Ctx& c, double* G, int layout, cudaStream_t s) {
  if (c.item1 <= c.item0) return cudaSuccess;
  cudaError_t e = cudaMemsetAsync(c.st.counter, 0, sizeof(unsigned long long), s);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  static bool attr_set = false;
  if (!attr_set) {
    e = cudaFuncSetAttribute(k_schur, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_schur, NT, kSmemBytes);
  per_sm = std::max(per_sm, 1);
  const int64_t want = std::min<int64_t>((int64_t)sms * per_sm, c.item1 - c.item0);
  SchurArgs a;
  a.arena = c.arena; a.ms = c.mstride; a.np = (int)c.np; a.n = (int)c.n; a.ncls = (int)c.ncls;
  a.npl = (int)c.npairs_local;
  a.cls_a = c.st.cls_a; a.cls_b = c.st.cls_b; a.pair_h = c.st.pair_h; a.pair_h2 = c.st.pair_h2;
  a.pair_kbeg = c.st.pair_kbeg; a.pair_item = c.st.pair_item; a.kL = c.st.k_L; a.kR = c.st.k_R;
  a.kf = c.st.k_flags; a.ks = c.st.k_scale; a.item0 = c.item0; a.item1 = c.item1; a.counter = c.st.counter;
  a.G = G; a.layout = layout; a.K = c.K; a.Ntil = c.Ntil;
  k_schur<<<(unsigned)want, NT, kSmemBytes, s>>>(a);
  ++c.launches;
  return cudaGetLastError();
}

}  // namespace polya
