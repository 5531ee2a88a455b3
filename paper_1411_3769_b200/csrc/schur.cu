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
// Work item = (pair, row class {i<=j}, column class {k<=l}) of 8-index chunks.  A CTA (160
// threads, 4 per SM) computes the <= 4 raw 64x64 sub-blocks of the item (one per orientation)
// with FP64 DMMA (mma.sync m8n8k4 -> DMMA.8x8x4; sm_100a has no f64 tcgen05 kind):
//  * a producer warp pulls items from an atomic counter (pair-major, so co-running CTAs share a
//    pair's operands in L2), one item ahead, and streams each orientation's k-list in stages of
//    8 terms (16 8x8 operand tiles, 16-byte cp.async) into a 2-slot mbarrier ring (tile stride
//    68 doubles: conflict-free fragment loads);
//  * 4 consumer warps split the valid M / N tiles 2 x 2 (4x4 DMMA tiles per warp, fewer for the
//    ragged last chunk of n, whose rows are packed two x-values per tile), fold each orientation
//    into a 32 KB XOR-swizzled shared G-block (conflict-free for all four orientations), ordered by
//    a phase mbarrier instead of CTA barriers, and write the item's G entries with table-driven,
//    diagonal-ordered (contiguous-run) stores plus mirror stores (FULL layout, diagonal pairs).
// Every G entry is produced by one CTA in a fixed k order: deterministic, and FULL layouts are
// bitwise symmetric.  DESIGN.md 5.2 has the measurements and the variants that were tried.
#include <algorithm>
#include <cassert>
#include <type_traits>

#include "polya_internal.h"

namespace polya {
namespace {

constexpr int Q = kChunk;  // 8
constexpr int KB = 8;      // k terms per pipeline stage (= kKStage: the k-lists are padded to whole stages)
static_assert(KB % 8 == 0 && kKStage % KB == 0, "stage size: two halves of whole k4 steps");
constexpr int NCW = 4;     // consumer (DMMA) warps: each a 4x4 grid of 8x8 tiles of the 64x64 sub-block
constexpr int NT = (NCW + 1) * 32;  // + one producer warp (cp.async into an mbarrier ring)
constexpr int NSTAGE = 2;  // ring depth: 2 slots so that 4 CTAs fit an SM (v20: 4 slots at 3 CTAs/SM, 2 % slower)
constexpr int kMinBlocks = 4;   // v23: 4 CTAs/SM (96 registers, a few spills outside the DMMA loop)
// Stage layout (v25): per operand (L, then R) 8 k-terms x 8 x 8 doubles, dense (4 KB).  Each tile is
// split into its 4 row pairs p = x >> 1 (128 bytes); k-term t's row pair p sits at byte
//   2048 (t >> 2) + 512 p + 128 (t & 3),   inside it row x & 1 at + 64, the 16-byte column pair
//   y >> 1 at + 16 ((y >> 1) ^ (t & 3)) (an XOR swizzle: the same pattern as TMA's 64-byte swizzle,
//   whose phase is address bits 7-8 = t & 3 here),
// so that (i) the 4 k-terms of a DMMA k-step and the 4 (x & 1, y & 1) rows of a half-warp's fragment
// loads hit 16 distinct bank slots, (ii) each producer copy instruction (one tile) fills 4 whole
// 128-byte bank rows, and (iii) a warp's M-tiles (which differ in p only, see orient<>) sit at constant
// 512-byte offsets: one address register per operand.  v24's padded 68-double tiles were conflict-free
// for the fragment loads only: its 544-byte tile starts made every cp.async take 2-3x the wavefronts.
constexpr int OPB = KB * 64 * 8;         // bytes per operand per stage (4096)
constexpr int STAGEB = 2 * OPB;          // bytes per stage (8192)
constexpr int STAGE = STAGEB / 8;        // doubles per stage
__host__ __device__ constexpr int stage_byte(int t, int x, int y) {
  return 2048 * (t >> 2) + 512 * (x >> 1) + 128 * (t & 3) + 64 * (x & 1) + 16 * ((y >> 1) ^ (t & 3)) + 8 * (y & 1);
}
// per slot: full (first half of the stage's k-terms landed), full2 (second half), empty (consumed)
constexpr size_t kSmemBytes = (NSTAGE * STAGE + Q * Q * Q * Q) * sizeof(double) + 3 * NSTAGE * sizeof(uint64_t);

#ifndef SCHUR_EXP
#define SCHUR_EXP 0   // tools-only timing variants (tools/schur_exp.py): 1 = no epilogue, 2 = no fold either,
                     // 4 = no mirror stores, 8 = item blocks stored contiguously (traffic experiments)
#endif                // (results wrong by construction: never a bench value)

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
  // optional schedule (full-range launches): pulled index -> item, pairs in decreasing k-list length
  // (longest items first: the last wave is made of short ones), a pair's items consecutive
  const int32_t* sched_pl;        // [nsched] local pair of schedule entry r
  const int64_t* sched_lo;        // [nsched] its first item in [item0, item1)
  const int64_t* sched_prefix;    // [nsched + 1] pulled-index prefix
  int nsched;
  unsigned long long* counter;
  double* G;
  double* const* tile_ptr;   // optional per-local-pair tile destination (the P2P combine: a peer's slot)
  int layout;
  int64_t K, Ntil;
  int64_t nmats;   // arena matrices (bounds checks of the POLYA_BOUNDS_CHECK build)
};

// Device-side bounds checks, compiled in only with -DPOLYA_BOUNDS_CHECK (compute-sanitizer is not
// available on this pool): arena matrix ids and G entries of every access are asserted in range.
#ifdef POLYA_BOUNDS_CHECK
#define POLYA_ASSERT(c) assert(c)
#else
#define POLYA_ASSERT(c) ((void)0)
#endif

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

// Shared G-block address of local (a,b,c,d): a GF(2)-linear bijection of the 12 coordinate bits onto
// [0, 4096), gs = Ta(a) ^ Tb(b) ^ Tc(c) ^ Td(d), each T a linear map of its 3 bits (columns below).
// 64-bit shared accesses are served per half-warp (16 lanes x 8 bytes = one 128-byte bank row), so the
// low 4 address bits (the 8-byte bank slot) must differ across the 16 lanes of each half of every
// fold store / load: for each orientation, the 4 coordinate bits that vary across a half-warp (x0, y0,
// w0, w1 with the tile rows of orient<>) have linearly independent low-4-bit columns (v24's swizzle
// met this for 4 of its 8 (orientation, packing) patterns only).
// Columns found by search; tests/test_layout_banks.py re-checks the folds, the bijection and bounds
// the epilogue's read conflicts.
__device__ __forceinline__ int lin3(int v, int c0, int c1, int c2) {
  return ((v & 1) ? c0 : 0) ^ ((v & 2) ? c1 : 0) ^ ((v & 4) ? c2 : 0);
}
__device__ __forceinline__ int Ta(int a) { return lin3(a, 11, 3, 10); }
__device__ __forceinline__ int Tb(int b) { return lin3(b, 7, 21, 32); }
__device__ __forceinline__ int Tc(int c) { return lin3(c, 65, 135, 264); }
__device__ __forceinline__ int Td(int d) { return lin3(d, 525, 1027, 2048); }

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gmem_src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(gmem_src));
}
__device__ __forceinline__ void st_g(double* p, double v) {
  POLYA_ASSERT(p != nullptr);
  *p = v;
}
__device__ __forceinline__ unsigned sptr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(sptr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}\n" ::"r"(sptr(bar)) : "memory");
}
// arrive-on triggered when all prior cp.async of this thread have completed (no pending-count change)
__device__ __forceinline__ void cp_async_mbar_arrive(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(sptr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(
          sptr(bar)),
      "r"(parity)
      : "memory");
}
// Consumer phases (each fold of an orientation, each item's epilogue) are ordered by one mbarrier
// with one arrival per consumer warp: a warp arrives when its part of a phase is done and waits
// for the previous phase only right before it touches Gs again, so a warp that finishes a fold
// early streams on into the next orientation's DMMAs instead of idling at a CTA barrier.
__device__ __forceinline__ void phase_arrive(uint64_t* bar, uint32_t& nph) {
  __syncwarp();
  if ((threadIdx.x & 31) == 0) mbar_arrive(bar);
  ++nph;
}
__device__ __forceinline__ void phase_wait_prev(uint64_t* bar, uint32_t nph) {
  if (nph > 0) mbar_wait(bar, (nph - 1) & 1);
}

struct ItemInfo {
  int pl, h, h2, sc, tc, ci, cj, ck, cl, nstage;
  int64_t kb;
};

// Item -> (pair, row class, column class).  `hint` is the pair of the CTA's previous item: items
// are pulled in increasing order, so the pair is usually the same or the next one (one load);
// otherwise a binary search.  Diagonal pairs enumerate classes sc <= tc row by row; the row is
// found in closed form (no O(ncls) loop).
__device__ __forceinline__ ItemInfo decode_item(const SchurArgs& p, int64_t item, int hint) {
  ItemInfo it;
  int lo = hint;
  if (!(lo >= 0 && lo < p.npl && __ldg(p.pair_item + lo) <= item && item < __ldg(p.pair_item + lo + 1))) {
    lo = 0;
    int hi = p.npl;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (__ldg(p.pair_item + mid) <= item) lo = mid; else hi = mid;
    }
  }
  it.pl = lo;
  it.h = __ldg(p.pair_h + lo);
  it.h2 = __ldg(p.pair_h2 + lo);
  const int64_t rem = item - __ldg(p.pair_item + lo);
  if (it.h != it.h2) {
    it.sc = (int)(rem / p.ncls);
    it.tc = (int)(rem - (int64_t)it.sc * p.ncls);
  } else {
    // row sc starts at st(sc) = sc*ncls - sc(sc-1)/2
    const int64_t N = p.ncls;
    const double N2 = 2.0 * (double)N + 1.0;
    int64_t sc = (int64_t)((N2 - sqrt(N2 * N2 - 8.0 * (double)rem)) * 0.5);
    sc = max((int64_t)0, min(sc, N - 1));
    while (sc > 0 && sc * N - sc * (sc - 1) / 2 > rem) --sc;
    while (sc + 1 < N && (sc + 1) * N - (sc + 1) * sc / 2 <= rem) ++sc;
    it.sc = (int)sc;
    it.tc = (int)(sc + rem - (sc * N - sc * (sc - 1) / 2));
  }
  it.ci = __ldg(p.cls_a + it.sc); it.cj = __ldg(p.cls_b + it.sc);
  it.ck = __ldg(p.cls_a + it.tc); it.cl = __ldg(p.cls_b + it.tc);
  it.kb = __ldg(p.pair_kbeg + lo);
  it.nstage = (int)((__ldg(p.pair_kbeg + lo + 1) - it.kb) / KB);   // k-lists are padded to whole stages
  return it;
}

// The item of pulled index idx (< item1 - item0): item0 + idx, or through the schedule, with the
// local pair as the decode hint (r: the schedule entry of the previous pull, tried first).
__device__ __forceinline__ int64_t sched_item(const SchurArgs& p, int64_t idx, int& hint, int& r) {
  if (!p.sched_prefix) return p.item0 + idx;
  if (!(r >= 0 && r < p.nsched && __ldg(p.sched_prefix + r) <= idx && idx < __ldg(p.sched_prefix + r + 1))) {
    int lo = 0, hi = p.nsched;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (__ldg(p.sched_prefix + mid) <= idx) lo = mid; else hi = mid;
    }
    r = lo;
  }
  hint = __ldg(p.sched_pl + r);
  return __ldg(p.sched_lo + r) + (idx - __ldg(p.sched_prefix + r));
}

// What the producer tells the consumers at the first stage of every item (and the end sentinel).
struct __align__(16) SlotInfo {
  long long item;
  int pl, h, h2, sc, tc, ci, cj, ck, cl, nstage;
};

// chunk roles of orientation o: Raw[(x,y),(z,w)] with x in cX, y in cY, z in cZ, w in cW; the
// local G index (a,b,c,d) is  o0: (w,x,y,z)  o1: (w,x,z,y)  o2: (x,w,y,z)  o3: (x,w,z,y)
template <class I>
__device__ __forceinline__ void roles(int o, const I& it, int& cX, int& cY, int& cZ, int& cW) {
  cX = (o & 2) ? it.ci : it.cj;
  cW = (o & 2) ? it.cj : it.ci;
  cY = (o & 1) ? it.cl : it.ck;
  cZ = (o & 1) ? it.ck : it.cl;
}

// One G entry of the item from the folded block: canonical summation order (direct, s-swap,
// t-swap, both) so that an entry and its mirror image are bitwise equal.  Table entries are
// {svec index, Gs term direct, Gs term swapped, has swap}.
template <bool DIAG>
__device__ __forceinline__ double gval(const double* Gs, int4 r, int4 c) {
  double v = Gs[r.y ^ c.y];
  if (DIAG) {   // only items with a diagonal class have swapped terms (no FP64 adds otherwise)
    if (r.w) v += Gs[r.z ^ c.y];
    if (c.w) v += Gs[r.y ^ c.z];
    if (r.w && c.w) v += Gs[r.z ^ c.z];
  }
  return v;
}

// One orientation of an item on the consumer warps: the raw sub-block
// Raw[(x,y),(z,w)] = sum_k L_k[x,y] R_k[z,w] (x in cX, y in cY, z in cZ, w in cW) over the
// item's nstage ring stages, then folded into Gs.  MMA rows are M-tiles (p, q) of 8 rows
// g -> (x, y) = (2p + (g & 1), 4q + (g >> 1)), columns N-tiles (p', q') the same way over (z, w).
// Full chunks: 8 M-tiles, warp row wm (of the 2 x 2 warp grid) takes q = wm, p = 0..3; a ragged x
// chunk (<= 4 valid x) needs p < 2 only (q = wm, p = 0..1), one with 5-6 valid x p < 3, a ragged y
// chunk (<= 4 valid y) q = 0 only (p = 2 wm + 0..1), both one tile (q = 0, p = wm) -- invalid rows
// (x, z) are never multiplied (a y / w chunk with 5-7 valid values keeps its q = 1 tiles whole).  A
// warp's tiles differ in p only, so their fragments sit at +512-byte steps of one lane offset.
template <int MI, int NJ, int RY, int RW>
__device__ __forceinline__ void orient(const SchurArgs& p, double* smem, double* Gs, uint64_t* full,
                                       uint64_t* empty, uint32_t& cnt, int nstage, int o, bool first,
                                       uint64_t* pbar, uint32_t& nph) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, t = lane & 3;
  const int wm = warp >> 1, wn = warp & 1;
  const int qm = RY ? 0 : wm, pm = RY ? MI * wm : 0;   // the warp's M-tiles: (pm + i, qm)
  const int qn = RW ? 0 : wn, pn = RW ? NJ * wn : 0;   // N-tiles: (pn + j, qn)
  // lane offsets (doubles, k-step 0, tile 0) of A[g][k=t] and B[k=t][n=g] in a stage
  const int oa = stage_byte(t, 2 * pm + (g & 1), 4 * qm + (g >> 1)) / 8;
  const int ob = (OPB + stage_byte(t, 2 * pn + (g & 1), 4 * qn + (g >> 1))) / 8;
  double acc[MI][NJ][2];
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NJ; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  for (int s = 0; s < nstage; ++s) {
    const uint32_t slot = cnt % NSTAGE, ph = (cnt / NSTAGE) & 1;
    mbar_wait(full + slot, ph);
    const double* fA = smem + slot * STAGE + oa;
    const double* fB = smem + slot * STAGE + ob;
#pragma unroll
    for (int k4 = 0; k4 < KB / 4; ++k4) {
      if (k4 == KB / 8) mbar_wait(full + 2 * NSTAGE + slot, ph);   // the stage's second half has landed
      double a[MI], b[NJ];
#pragma unroll
      for (int i = 0; i < MI; ++i) a[i] = fA[k4 * 256 + i * 64];   // + 2048 bytes per k-step, 512 per tile
#pragma unroll
      for (int j = 0; j < NJ; ++j) b[j] = fB[k4 * 256 + j * 64];
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NJ; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + slot);
    ++cnt;
  }
  if (SCHUR_EXP & 2) {   // timing experiment: no fold, no epilogue (a never-taken sink keeps the DMMAs)
    double sum = 0.0;
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
      for (int j = 0; j < NJ; ++j) sum += acc[i][j][0] * acc[i][j][1];
    if (sum == 1.2345e-300) p.G[tid] = sum;
    return;
  }
  phase_wait_prev(pbar, nph);   // the previous fold / the previous item's epilogue is done with Gs
  // fold: acc[i][j][e] = Raw(x, y, z, w) -> Gs[(a,b,c,d)(o)], gs = Ta(a)^Tb(b)^Tc(c)^Td(d) split into
  // per-coordinate terms: x -> (o&2 ? Ta : Tb), w -> (o&2 ? Tb : Ta), y -> (o&1 ? Td : Tc),
  // z -> (o&1 ? Tc : Td)   (o0: (a,b,c,d) = (w,x,y,z), o1: (w,x,z,y), o2: (x,w,y,z), o3: (x,w,z,y));
  // accumulator column 2t+e of N-tile (p', q') is (z, w) = (2p' + e, 4q' + t)
  int bx[MI], bz[NJ][2];
#pragma unroll
  for (int i = 0; i < MI; ++i) {
    const int x = 2 * (pm + i) + (g & 1), y = 4 * qm + (g >> 1);
    bx[i] = ((o & 2) ? Ta(x) : Tb(x)) ^ ((o & 1) ? Td(y) : Tc(y));
  }
#pragma unroll
  for (int j = 0; j < NJ; ++j)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int z = 2 * (pn + j) + e, w = 4 * qn + t;
      bz[j][e] = ((o & 1) ? Tc(z) : Td(z)) ^ ((o & 2) ? Tb(w) : Ta(w));
    }
  if (first) {
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
      for (int j = 0; j < NJ; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) Gs[bx[i] ^ bz[j][e]] = acc[i][j][e];
  } else {
#pragma unroll
    for (int i = 0; i < MI; ++i) {  // 2*NJ independent read-modify-writes at a time
      double old[NJ][2];
#pragma unroll
      for (int j = 0; j < NJ; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) old[j][e] = Gs[bx[i] ^ bz[j][e]];
#pragma unroll
      for (int j = 0; j < NJ; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) Gs[bx[i] ^ bz[j][e]] = old[j][e] + acc[i][j][e];
    }
  }
  phase_arrive(pbar, nph);
}

// (M side, N side) code -> instantiation: code 0: 8 tiles (4 per warp), 1: 4 tiles of a ragged x / z
// chunk, 2: 4 tiles of a ragged y / w chunk, 3: 2 tiles (both ragged), 4: 6 tiles of an x / z chunk
// with 5-6 valid values (p < 3: rows x = 6, 7 are never formed).
#define ORIENT_M(MC, MI, RY)                                                                          \
  case MC * 5 + 0: orient<MI, 4, RY, 0>(p, smem, Gs, full, empty, cnt, nstage, o, first, pbar, nph); break; \
  case MC * 5 + 1: orient<MI, 2, RY, 0>(p, smem, Gs, full, empty, cnt, nstage, o, first, pbar, nph); break; \
  case MC * 5 + 2: orient<MI, 2, RY, 1>(p, smem, Gs, full, empty, cnt, nstage, o, first, pbar, nph); break; \
  case MC * 5 + 3: orient<MI, 1, RY, 1>(p, smem, Gs, full, empty, cnt, nstage, o, first, pbar, nph); break; \
  case MC * 5 + 4: orient<MI, 3, RY, 0>(p, smem, Gs, full, empty, cnt, nstage, o, first, pbar, nph); break;
__device__ __forceinline__   // inlined: the out-of-line call cost 1.7 ms (cfg 4) and 34 ms (cfg 5)
void orient_dispatch(int code, const SchurArgs& p, double* smem, double* Gs, uint64_t* full,
                                             uint64_t* empty, uint32_t& cnt, int nstage, int o, bool first,
                                             uint64_t* pbar, uint32_t& nph) {
  switch (code) {
    ORIENT_M(0, 4, 0)
    ORIENT_M(1, 2, 0)
    ORIENT_M(2, 2, 1)
    ORIENT_M(3, 1, 1)
    ORIENT_M(4, 3, 0)
  }
}
#undef ORIENT_M

__global__ void __launch_bounds__(NT, kMinBlocks) k_schur(const SchurArgs p) {
  extern __shared__ __align__(16) double smem[];
  double* Gs = smem + NSTAGE * STAGE;
  uint64_t* full = reinterpret_cast<uint64_t*>(Gs + Q * Q * Q * Q);   // first half landed (32 + 1 arrivals)
  uint64_t* empty = full + NSTAGE;                                      // stage consumed (NCW arrivals)
  // full + 2 NSTAGE: second half landed (32 cp.async arrivals)
  __shared__ unsigned char s_diag[64][2];  // (lc, ld) of local pairs ordered by (ld-lc, lc)
  __shared__ int4 s_rt[2][64], s_ct[2][64];   // epilogue tables of the item's valid row / column pairs
  __shared__ int s_nrc[2][2];                  // their counts (double-buffered by item parity)
  __shared__ uint64_t s_pbar;                  // consumer phase barrier (NCW arrivals per phase)
  __shared__ SlotInfo s_info[NSTAGE];      // item of the stage held by each ring slot (first stages)
  __shared__ SlotInfo s_cur[NCW];          // each consumer warp's current item

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid < 64) {  // diagonal order: consecutive entries have consecutive svec indices
    int idx = 0;
    for (int dlt = -(Q - 1); dlt <= Q - 1; ++dlt)
      for (int lc = max(0, -dlt); lc <= min(Q - 1, Q - 1 - dlt); ++lc, ++idx)
        if (idx == tid) { s_diag[tid][0] = (unsigned char)lc; s_diag[tid][1] = (unsigned char)(lc + dlt); }
  }
  if (tid == 0) {
    for (int i = 0; i < NSTAGE; ++i) {
      mbar_init(full + i, 33);   // 32 cp.async completions + lane 0's release of s_info
      mbar_init(full + 2 * NSTAGE + i, 32);   // the second half's completions
      mbar_init(empty + i, NCW);
    }
    mbar_init(&s_pbar, NCW);
  }
  __syncthreads();
  const int n = p.n, np = p.np;

  // Dynamic schedule: the producer pulls items from an atomic counter (pair-major order, so
  // co-running CTAs share a pair's operands in L2), one item ahead: while it streams item i it
  // already holds the index, decode and first k-descriptors of item i+1, so no stage waits on
  // an atomic, a table lookup or a descriptor load.  The consumers learn each item from s_info.
  if (warp == NCW) {
    // ===== producer warp: 16-byte cp.async chunks (row sr, column pair sc2) of all 16 tiles into
    // the swizzled stage layout (stage_byte) =====
    const int sr = lane >> 2, sc2 = lane & 3;
    uint32_t cnt = 0;
    unsigned long long got = 0;
    const int64_t total = p.item1 - p.item0;
    int sr_ = -1, hint = -1;   // schedule entry and pair of the last pull
    if (lane == 0) got = atomicAdd(p.counter, 1ULL);
    int64_t idx = (int64_t)__shfl_sync(0xffffffffu, got, 0);
    int64_t item = idx < total ? sched_item(p, idx, hint, sr_) : p.item1;
    ItemInfo it{};
    int2 dfirst = make_int2(0, 0);
    if (item < p.item1) {
      it = decode_item(p, item, hint);
      if (lane < KB) dfirst = __ldg(p.kdesc + it.kb + lane);
      if (lane == 0) got = atomicAdd(p.counter, 1ULL);
    }
    while (item < p.item1) {
      // next item: index (requested one item ago), decode and first descriptors, in flight now
      const int64_t idx_n = (int64_t)__shfl_sync(0xffffffffu, got, 0);
      int hint_n = it.pl;
      const int64_t item_n = idx_n < total ? sched_item(p, idx_n, hint_n, sr_) : p.item1;
      ItemInfo it_n{};
      int2 dfirst_n = make_int2(0, 0);
      if (item_n < p.item1) {
        it_n = decode_item(p, item_n, hint_n);
        if (lane < KB) dfirst_n = __ldg(p.kdesc + it_n.kb + lane);
        if (lane == 0) got = atomicAdd(p.counter, 1ULL);
      }
      const bool dS = (it.ci == it.cj), dT = (it.ck == it.cl);
      bool first_stage = true;
      for (int o = 0; o < 4; ++o) {
        if ((o & 1) && dT) continue;
        if ((o & 2) && dS) continue;
        int cX, cY, cZ, cW;
        roles(o, it, cX, cY, cZ, cW);
        const int offL = (cX * Q + sr) * np + cY * Q + 2 * sc2;
        const int offR = (cZ * Q + sr) * np + cW * Q + 2 * sc2;
        int2 dcur = dfirst;
        for (int s = 0; s < it.nstage; ++s) {
          // descriptors of the next stage: the next k-block, or the first one again (the next
          // orientation walks the same k-list; the next item's were loaded above)
          int2 dnext = dfirst;
          if (s + 1 < it.nstage && lane < KB) dnext = __ldg(p.kdesc + it.kb + (int64_t)(s + 1) * KB + lane);
          const uint32_t slot = cnt % NSTAGE, ph = (cnt / NSTAGE) & 1;
          mbar_wait(empty + slot, ph ^ 1);
          if (first_stage && lane == 0) {
            SlotInfo si;
            si.item = item; si.pl = it.pl; si.h = it.h; si.h2 = it.h2; si.sc = it.sc; si.tc = it.tc;
            si.ci = it.ci; si.cj = it.cj; si.ck = it.ck; si.cl = it.cl; si.nstage = it.nstage;
            s_info[slot] = si;
          }
          first_stage = false;
          char* T = reinterpret_cast<char*>(smem + slot * STAGE);
#pragma unroll
          for (int kk = 0; kk < KB; ++kk) {
            const unsigned idL = (unsigned)__shfl_sync(0xffffffffu, dcur.x, kk);
            const unsigned idR = (unsigned)__shfl_sync(0xffffffffu, dcur.y, kk);
            POLYA_ASSERT(idL < p.nmats && idR < p.nmats);
            const int db = stage_byte(kk, sr, 2 * sc2);
            cp_async16(T + db, p.arena + (uint64_t)idL * p.ms32 + offL);
            cp_async16(T + OPB + db, p.arena + (uint64_t)idR * p.ms32 + offR);
            if (kk == KB / 2 - 1) {   // first half of the k-terms: consumers may start on it
              cp_async_mbar_arrive(full + slot);
              if (lane == 0) mbar_arrive(full + slot);   // releases s_info[slot]
            }
          }
          cp_async_mbar_arrive(full + 2 * NSTAGE + slot);
          dcur = dnext;
          ++cnt;
        }
      }
      item = item_n;
      it = it_n;
      dfirst = dfirst_n;
    }
    {  // end-of-work sentinel stage
      const uint32_t slot = cnt % NSTAGE, ph = (cnt / NSTAGE) & 1;
      mbar_wait(empty + slot, ph ^ 1);
      if (lane == 0) s_info[slot].item = p.item1;
      cp_async_mbar_arrive(full + slot);
      if (lane == 0) mbar_arrive(full + slot);
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    return;
  }

  // ===== consumer warps: DMMA on ring stages, fold into Gs, epilogue ==========================
  uint32_t cnt = 0, nph = 0;
  int icount = 0;
  for (;;) {
    {  // the next ring stage is the first stage of the next item (or the end sentinel)
      const uint32_t slot = cnt % NSTAGE, ph = (cnt / NSTAGE) & 1;
      mbar_wait(full + slot, ph);
    }
    // the item's descriptor stays in shared memory (a per-warp copy: the ring slot's s_info may be
    // rewritten for a later item while this one is still folding / writing), read where it is used,
    // so that it holds no registers across the DMMA loops
    if (lane == 0) s_cur[warp] = s_info[cnt % NSTAGE];
    __syncwarp();
    const volatile SlotInfo& it = s_cur[warp];
    if (it.item >= p.item1) {
      if (p.tile_ptr) __threadfence_system();   // P2P combine: the stores to peer memory before the signal
      break;
    }
    const bool dS = (it.ci == it.cj), dT = (it.ck == it.cl);
    const int tb = icount & 1;
    ++icount;
    // Tables of the item's valid local pairs (buffer tb: its previous user, item i-2, finished
    // its epilogue before item i-1's first fold), compacted in diagonal order (consecutive
    // entries have consecutive svec indices, so a warp's stores form contiguous runs): warp 0
    // the rows (a,b) of class (ci,cj), warp 1 the columns (c,d) of class (ck,cl).  Published to
    // the other warps by the fold-phase arrivals.
    if (warp < 2 && !(SCHUR_EXP & 3)) {
      const bool rows = (warp == 0);
      const int c1 = rows ? it.ci : it.ck, c2 = rows ? it.cj : it.cl;
      const bool dg = rows ? dS : dT;
      int4* tab = rows ? s_rt[tb] : s_ct[tb];
      int base = 0;
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        const int q = lane + 32 * half;
        const int u1 = s_diag[q][0], u2 = s_diag[q][1];
        const int A = c1 * Q + u1, B = c2 * Q + u2;
        const bool valid = (A < n) && (B < n) && (!dg || u1 <= u2);
        const unsigned bal = __ballot_sync(0xffffffffu, valid);
        if (valid) {
          const int pos = base + __popc(bal & ((1u << lane) - 1u));
          tab[pos] = rows ? make_int4((int)svec_idx(A, B, n), Ta(u1) ^ Tb(u2), Ta(u2) ^ Tb(u1), dg && u1 != u2)
                          : make_int4((int)svec_idx(A, B, n), Tc(u1) ^ Td(u2), Tc(u2) ^ Td(u1), dg && u1 != u2);
        }
        base += __popc(bal);
      }
      if (lane == 0) s_nrc[tb][warp] = base;
    }
    bool first = true;
    for (int o = 0; o < 4; ++o) {
      if ((o & 1) && dT) continue;
      if ((o & 2) && dS) continue;
      int cX, cY, cZ, cW;
      roles(o, it, cX, cY, cZ, cW);
      // ragged chunk (n not a multiple of 8) in an MMA dimension (y: M rows, w: N columns): with
      // <= 4 valid indices, pack two x (or z) values into one 8-row MMA tile instead of
      // multiplying 8-row tiles that are half zeros
      const bool rY = (n - cY * Q) <= 4, rW = (n - cW * Q) <= 4;   // packed MMA rows / columns
      const bool rX = (n - cX * Q) <= 4, rZ = (n - cZ * Q) <= 4;   // only 4 x (z) values exist
      const bool sX = (n - cX * Q) <= 6, sZ = (n - cZ * Q) <= 6;   // only 6: x (z) = 6, 7 never formed
      const int mcode = rY ? (rX ? 3 : 2) : (rX ? 1 : (sX ? 4 : 0));
      const int ncode = rW ? (rZ ? 3 : 2) : (rZ ? 1 : (sZ ? 4 : 0));
      orient_dispatch(mcode * 5 + ncode, p, smem, Gs, full, empty, cnt, it.nstage, o, first, &s_pbar, nph);
      first = false;
    }
    if (SCHUR_EXP & 3) continue;   // timing experiment: no epilogue
    phase_wait_prev(&s_pbar, nph);   // all folds of the item are in Gs (and its tables are written)
    // ---- epilogue: fold diagonal classes and write G ----------------------------------------
    const int nr = s_nrc[tb][0], nc = s_nrc[tb][1];
    const bool diag_pair = (it.h == it.h2);
    const bool same_cls = diag_pair && (it.sc == it.tc);
    const bool fullG = (p.layout == POLYA_G_FULL);
    const int64_t rowbase = (int64_t)it.h * p.Ntil, colbase = (int64_t)it.h2 * p.Ntil;
    double* tile = p.tile_ptr ? p.tile_ptr[it.pl] : p.G + (int64_t)it.pl * p.Ntil * p.Ntil;
    const int4 none = make_int4(-1, 0, 0, 0);
    auto passes = [&](auto diag_tag) {
      constexpr bool DIAG = decltype(diag_tag)::value;
    {  // pass 0: direct entries G[s][t], lanes along the columns t; 4 rows per warp in flight
      const int4 cA = lane < nc ? s_ct[tb][lane] : none, cB = lane + 32 < nc ? s_ct[tb][lane + 32] : none;
      for (int r0 = warp; r0 < nr; r0 += 4 * NCW) {
        int4 rw[4];
        double vA[4], vB[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) rw[u] = r0 + u * NCW < nr ? s_rt[tb][r0 + u * NCW] : none;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          vA[u] = (rw[u].x >= 0 && cA.x >= 0) ? gval<DIAG>(Gs, rw[u], cA) : 0.0;
          vB[u] = (rw[u].x >= 0 && cB.x >= 0) ? gval<DIAG>(Gs, rw[u], cB) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (rw[u].x < 0) continue;
          POLYA_ASSERT(rw[u].x < p.Ntil && cA.x < p.Ntil && cB.x < p.Ntil && it.pl < p.npl);
          double* dst = fullG ? p.G + (rowbase + rw[u].x) * p.K + colbase : tile + (int64_t)rw[u].x * p.Ntil;
          if (SCHUR_EXP & 8) {   // traffic experiment: the item's block contiguous (whole sectors), wrong G
            const int64_t span = (int64_t)p.npl * p.Ntil * p.Ntil - 4096;
            double* blk = p.G + (int64_t)(((unsigned long long)it.item * 4096ull) % (unsigned long long)span);
            if (cA.x >= 0) st_g(blk + (r0 + u * NCW) * 64 + lane, vA[u]);
            if (cB.x >= 0) st_g(blk + (r0 + u * NCW) * 64 + lane + 32, vB[u]);
            continue;
          }
          if (cA.x >= 0 && !(same_cls && rw[u].x > cA.x)) st_g(dst + cA.x, vA[u]);
          if (cB.x >= 0 && !(same_cls && rw[u].x > cB.x)) st_g(dst + cB.x, vB[u]);
        }
      }
    }
    if ((fullG || diag_pair) && !(SCHUR_EXP & 12)) {  // pass 1: mirror entries G[t][s], lanes along the rows s
      const int4 rA = lane < nr ? s_rt[tb][lane] : none, rB = lane + 32 < nr ? s_rt[tb][lane + 32] : none;
      for (int c0 = warp; c0 < nc; c0 += 4 * NCW) {
        int4 cl[4];
        double vA[4], vB[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) cl[u] = c0 + u * NCW < nc ? s_ct[tb][c0 + u * NCW] : none;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          vA[u] = (cl[u].x >= 0 && rA.x >= 0) ? gval<DIAG>(Gs, rA, cl[u]) : 0.0;
          vB[u] = (cl[u].x >= 0 && rB.x >= 0) ? gval<DIAG>(Gs, rB, cl[u]) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (cl[u].x < 0) continue;
          POLYA_ASSERT(cl[u].x < p.Ntil && rA.x < p.Ntil && rB.x < p.Ntil && it.pl < p.npl);
          double* dst = fullG ? p.G + (colbase + cl[u].x) * p.K + rowbase : tile + (int64_t)cl[u].x * p.Ntil;
          if (rA.x >= 0 && !(same_cls && rA.x > cl[u].x)) st_g(dst + rA.x, vA[u]);
          if (rB.x >= 0 && !(same_cls && rB.x > cl[u].x)) st_g(dst + rB.x, vB[u]);
        }
      }
    }
    };
    if (dS || dT) passes(std::true_type{});
    else passes(std::false_type{});
    phase_arrive(&s_pbar, nph);   // this warp is done reading Gs for the item
  }
}

}  // namespace

cudaError_t launch_schur(Ctx& c, double* G, int layout, int64_t i0, int64_t i1, cudaStream_t s, double* const* tile_ptr) {
  if (i1 <= i0) return cudaSuccess;
  cudaError_t e = cudaMemsetAsync(c.st.counter, 0, sizeof(unsigned long long), s);
  if (e != cudaSuccess) return e;
  if (c.k4_ctas == 0) {   // once per context: shared-memory attribute and resident CTAs (persistent grid)
    e = cudaFuncSetAttribute(k_schur, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes);
    if (e != cudaSuccess) return e;
    int sms = 0, per_sm = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c.device);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_schur, NT, kSmemBytes);
    c.k4_ctas = (int64_t)sms * std::max(per_sm, 1);
  }
  const int64_t want = std::min<int64_t>(c.k4_ctas, i1 - i0);
  SchurArgs a;
  a.arena = c.arena; a.ms = c.mstride; a.ms32 = (unsigned)c.mstride; a.np = (int)c.np; a.n = (int)c.nbas; a.ncls = (int)c.ncls;
  a.npl = (int)c.npairs_local;
  a.cls_a = c.st.cls_a; a.cls_b = c.st.cls_b; a.pair_h = c.st.pair_h; a.pair_h2 = c.st.pair_h2;
  a.pair_kbeg = c.st.pair_kbeg; a.pair_item = c.st.pair_item; a.kdesc = c.st.kdesc;
  a.item0 = i0; a.item1 = i1; a.counter = c.st.counter;
  // the whole share with few items per CTA (config 3; a rank's share at N = 8): longest items first, so the
  // last wave is made of short ones.  With hundreds of items per CTA the tail is negligible and the
  // pair-major order's L2 reuse across neighbouring pairs wins (config 5: +1.2 % with the schedule).
  const bool full = i0 == c.item0 && i1 == c.item1 && c.st.nsched > 0 && (i1 - i0) < 128 * c.k4_ctas;
  a.sched_pl = full ? c.st.sched_pl : nullptr;
  a.sched_lo = full ? c.st.sched_lo : nullptr;
  a.sched_prefix = full ? c.st.sched_prefix : nullptr;
  a.nsched = full ? (int)c.st.nsched : 0;
  a.G = G; a.tile_ptr = tile_ptr; a.layout = layout; a.K = c.K; a.Ntil = c.Ntil; a.nmats = c.nmats;
  k_schur<<<(unsigned)want, NT, kSmemBytes, s>>>(a);
  ++c.launches;
  return cudaGetLastError();
}

}  // namespace polya
