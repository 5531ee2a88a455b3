// polya_host.cpp -- host side of the C ABI (include/polya.h): Algorithm 1's set-up
// re-designed for one B200 per rank, plus the entry points that
// marshal device pointers into the kernels of kernels.cu / schur.cu / ipm.cu.
//
// Set-up uses the closed forms of the Polya coefficients:
//   beta_{h,gamma} = multinomial(d1; gamma - h)                        (Eq. beta)
//   H_{h,gamma}    = sum_{lambda in W_da} multinomial(d2; gamma-h-lambda) A_lambda  (Eq. H, 226-235)
//   c_gamma        = delta * multinomial(dp + d1; gamma)               (Eq. Cj, 347-351)
// which equal the paper's recursions (each recursion step is one multiplication by
// sum_i alpha_i, so d steps give the multinomial expansion of (sum_i alpha_i)^d).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <new>

#include "polya_internal.h"

using namespace polya;

namespace {

struct Fail {
  polya_status s;
  std::string msg;
};

#define CU(x)                                                                                   \
  do {                                                                                          \
    cudaError_t e_ = (x);                                                                       \
    if (e_ != cudaSuccess) throw Fail{POLYA_ECUDA, std::string(#x) + ": " + cudaGetErrorString(e_)}; \
  } while (0)

int64_t mul_chk(int64_t a, int64_t b) {
  int64_t r;
  if (__builtin_mul_overflow(a, b, &r)) throw Fail{POLYA_EOVERFLOW, "int64 overflow"};
  return r;
}
int64_t add_chk(int64_t a, int64_t b) {
  int64_t r;
  if (__builtin_add_overflow(a, b, &r)) throw Fail{POLYA_EOVERFLOW, "int64 overflow"};
  return r;
}

// C(nn, kk), checked.
int64_t binom(int64_t nn, int64_t kk) {
  if (kk < 0 || kk > nn) return 0;
  kk = std::min(kk, nn - kk);
  __int128 r = 1;
  for (int64_t i = 0; i < kk; ++i) {
    r = r * (nn - i) / (i + 1);
    if (r > (__int128)INT64_MAX) throw Fail{POLYA_EOVERFLOW, "binomial overflow"};
  }
  return (int64_t)r;
}

// Eq. (2): f(l, d) = C(l + d - 1, l - 1), 0 for l = 0.
int64_t card(int64_t l, int64_t d) { return l == 0 ? 0 : binom(add_chk(l, d) - 1, l - 1); }

// multinomial(d; parts) = prod_i C(p_1 + .. + p_i, p_i); 0 if a part is negative or sum != d.
int64_t multinomial(int64_t d, const int32_t* parts, int64_t l) {
  int64_t s = 0, r = 1;
  for (int64_t i = 0; i < l; ++i) {
    if (parts[i] < 0) return 0;
    s += parts[i];
    r = mul_chk(r, binom(s, parts[i]));
  }
  return s == d ? r : 0;
}

// W_d in the prose order of PAPER.md:58 (reading R1): descending lexicographic.
void enumerate(int64_t l, int64_t d, std::vector<int32_t>& out) {
  out.clear();
  std::vector<int32_t> cur(l, 0);
  // recursive descent: position i takes values from `rem` down to 0
  struct Rec {
    static void go(int64_t i, int64_t l, int64_t rem, std::vector<int32_t>& cur, std::vector<int32_t>& out) {
      if (i == l - 1) {
        cur[i] = (int32_t)rem;
        out.insert(out.end(), cur.begin(), cur.end());
        return;
      }
      for (int64_t v = rem; v >= 0; --v) {
        cur[i] = (int32_t)v;
        go(i + 1, l, rem - v, cur, out);
      }
    }
  };
  Rec::go(0, l, d, cur, out);
}

template <class T>
T* dalloc(int64_t count) {
  if (count <= 0) return nullptr;
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, (size_t)count * sizeof(T));
  if (e != cudaSuccess) {
    cudaGetLastError();
    throw Fail{POLYA_ENOMEM, std::string("cudaMalloc: ") + cudaGetErrorString(e)};
  }
  return (T*)p;
}
template <class T>
T* dupload(const std::vector<T>& v) {
  T* p = dalloc<T>((int64_t)v.size());
  if (p) CU(cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
  return p;
}

// K3b descriptors of one precompute launch: the groups, their entries and the 64-row tiles of each group.
void rg_upload(Ctx& c, int phase, const std::vector<RgGroup>& grp, const std::vector<RgEnt>& ent) {
  std::vector<RgTile> tiles;
  for (size_t g = 0; g < grp.size(); ++g) {
    const int64_t rows = (int64_t)(grp[g].eend - grp[g].ebeg) * c.np;
    if (rows > INT32_MAX) throw Fail{POLYA_EOVERFLOW, "precompute group too large"};
    for (int64_t r0 = 0; r0 < rows; r0 += 64) tiles.push_back({(int32_t)g, (int32_t)r0});
  }
  c.d_rg_grp[phase] = dupload(grp);
  c.d_rg_ent[phase] = dupload(ent);
  c.d_rg_tile[phase] = dupload(tiles);
  c.n_rg_tile[phase] = (int64_t)tiles.size();
}

// The generalised form's input terms (polya_setup_general, reading R18).
struct GenInput {
  int32_t nterms;
  const int32_t *deg_a, *deg_b;
  const double *At, *Bt, *R;
  int32_t N;   // block order (>= cfg.n; N > n: At_i is N x n, Bt_i n x N, R N x N)
};

void build(Ctx& c, const double* A_host, bool device = true, const GenInput* gi = nullptr) {
  const polya_config& g = c.cfg;
  c.nbas = g.n;
  c.n = (gi && gi->N > g.n) ? gi->N : g.n;
  c.l = g.l;
  c.L0 = card(g.l, g.dp);
  c.L = card(g.l, (int64_t)g.dp + g.d1);
  c.M = card(g.l, (int64_t)g.dp + g.da + g.d2);
  c.nA = card(g.l, g.da);
  c.nb = add_chk(c.L, c.M);
  c.Ntil = mul_chk(c.nbas, c.nbas + 1) / 2;
  c.K = mul_chk(c.L0, c.Ntil);
  (void)mul_chk(c.K, c.K);  // K*K must be representable (FULL layout indexing)
  c.np = (c.n + kChunk - 1) / kChunk * kChunk;
  c.r = (c.nbas + kChunk - 1) / kChunk;   // index chunks of the basis (K4 work items)
  c.ncls = c.r * (c.r + 1) / 2;
  c.mstride = mul_chk(c.np, c.np);
  if (c.mstride >= (int64_t)1 << 31) throw Fail{POLYA_EOVERFLOW, "n too large for 32-bit tile offsets"};
  const int64_t l = c.l;

  enumerate(l, g.dp, c.Wp);
  enumerate(l, (int64_t)g.dp + g.d1, c.WL);
  enumerate(l, (int64_t)g.dp + g.da + g.d2, c.WM);
  enumerate(l, g.da, c.Wa);
  if ((int64_t)c.Wp.size() != c.L0 * l || (int64_t)c.WL.size() != c.L * l ||
      (int64_t)c.WM.size() != c.M * l || (int64_t)c.Wa.size() != c.nA * l)
    throw Fail{POLYA_EOVERFLOW, "enumeration size mismatch"};

  // beta (Eq. beta) and C (Eq. Cj)
  std::vector<int32_t> tmp(l);
  c.beta.assign(c.L0 * c.L, 0);
  c.c.assign(c.L, 0.0);
  c.nnz_beta = 0;
  for (int64_t j = 0; j < c.L; ++j) {
    const int32_t* gj = &c.WL[j * l];
    for (int64_t h = 0; h < c.L0; ++h) {
      for (int64_t i = 0; i < l; ++i) tmp[i] = gj[i] - c.Wp[h * l + i];
      int64_t b = multinomial(g.d1, tmp.data(), l);
      c.beta[h * c.L + j] = b;
      if (b) ++c.nnz_beta;
    }
    c.c[j] = g.delta * (double)multinomial((int64_t)g.dp + g.d1, gj, l);
  }
  // nonzero beta entries (h, j) -> e (h-major): slots of the pre-scaled copies beta_hj X_j, beta_hj W_j
  std::vector<int32_t> bidx(c.L0 * c.L, -1);
  std::vector<int32_t> be_src;
  std::vector<double> be_w;
  for (int64_t h = 0; h < c.L0; ++h)
    for (int64_t j = 0; j < c.L; ++j)
      if (c.beta[h * c.L + j]) {
        bidx[h * c.L + j] = (int32_t)be_src.size();
        be_src.push_back((int32_t)j);
        be_w.push_back((double)c.beta[h * c.L + j]);
      }
  // nonzero H entries (h, m), m-major, with their integer weights per lambda
  c.Hidx.assign(c.L0 * c.M, -1);
  c.Hcnt.assign(c.L0 * c.M, 0);
  c.Hh.clear(); c.Hm.clear(); c.Hw.clear();
  std::vector<double> w(c.nA);
  // generalised form: term t = (A_t, B_t) as weighted sums of coefficient matrices (src, weight)
  std::vector<std::vector<std::pair<int32_t, double>>> tA, tB;
  std::vector<double> coefN;   // generalised form: the terms' coefficients padded to N x N
  c.gen = gi != nullptr;
  if (c.gen) {
    // coefficient layout: pair i's At coefficients (W_{a_i} order), then its Bt coefficients
    std::vector<std::vector<int32_t>> Wa_i(gi->nterms), Wb_i(gi->nterms);
    c.gp_da.assign(gi->deg_a, gi->deg_a + gi->nterms);
    c.gp_db.assign(gi->deg_b, gi->deg_b + gi->nterms);
    c.gp_aoff.clear(); c.gp_boff.clear(); c.coef_exp.clear();
    int64_t off = 0;
    for (int32_t i = 0; i < gi->nterms; ++i) {
      enumerate(l, c.gp_da[i], Wa_i[i]);
      enumerate(l, c.gp_db[i], Wb_i[i]);
      c.gp_aoff.push_back((int32_t)off);
      off += (int64_t)Wa_i[i].size() / l;
      c.gp_boff.push_back((int32_t)off);
      off += (int64_t)Wb_i[i].size() / l;
      c.coef_exp.insert(c.coef_exp.end(), Wa_i[i].begin(), Wa_i[i].end());
      c.coef_exp.insert(c.coef_exp.end(), Wb_i[i].begin(), Wb_i[i].end());
    }
    c.r_off = off;
    c.r_cnt = 0;
    // every coefficient as an N x N matrix (At: N x n in the left columns, Bt: n x N in the top rows,
    // zero elsewhere -- reading R19), and canonical ids: bitwise-equal coefficient matrices (an
    // identity repeated per vertex, say) share the smallest id, so the merges below see one matrix
    const int64_t NB = c.n, nbs = c.nbas, NN = NB * NB;
    coefN.assign((size_t)off * NN, 0.0);
    {
      int64_t ua = 0, ub = 0;
      for (int32_t i = 0; i < gi->nterms; ++i) {
        for (int64_t q = c.gp_aoff[i]; q < c.gp_boff[i]; ++q, ++ua)
          for (int64_t r = 0; r < NB; ++r)
            for (int64_t col = 0; col < nbs; ++col) coefN[q * NN + r * NB + col] = gi->At[(ua * NB + r) * nbs + col];
        const int64_t bend = i + 1 < gi->nterms ? c.gp_aoff[i + 1] : off;
        for (int64_t q = c.gp_boff[i]; q < bend; ++q, ++ub)
          for (int64_t r = 0; r < nbs; ++r)
            for (int64_t col = 0; col < NB; ++col) coefN[q * NN + r * NB + col] = gi->Bt[(ub * nbs + r) * NB + col];
      }
    }
    std::vector<int32_t> canon(off);
    for (int64_t q = 0; q < off; ++q) {
      canon[q] = (int32_t)q;
      for (int64_t r = 0; r < q; ++r)
        if (canon[r] == r && std::memcmp(&coefN[q * NN], &coefN[r * NN], (size_t)NN * sizeof(double)) == 0) {
          canon[q] = (int32_t)r;
          break;
        }
    }
    if (gi->R) {   // the constant term: coefficients in W_{dp+da} order (verdict) and C on Lyapunov blocks
      std::vector<int32_t> Wr;
      enumerate(l, (int64_t)g.dp + g.da, Wr);
      c.r_cnt = (int64_t)Wr.size() / l;
      off += c.r_cnt;
      c.coef_exp.insert(c.coef_exp.end(), Wr.begin(), Wr.end());
    }
    c.ncoef = off;
    // block gamma_m of element (h, k): -sum_{i, lambda, mu} multinomial(d2; gamma - h - lambda - mu)
    //   (At_{i,lambda} E_k Bt_{i,mu} + transpose); the sum over the larger of W_{a_i}, W_{b_i} is folded
    //   into one weighted coefficient sum, so (h, m) gets min(f(l,a_i), f(l,b_i)) terms per i at most
    // Exact term merges per (h, gamma) (the weights are integers): a side that is one coefficient
    // matrix times a weight takes the weight over to the other side; terms whose B side is the same
    // single matrix then merge by adding their A sides (A E B + A' E B = (A + A') E B), and likewise
    // for a shared single A side.  Discrete time's (-1/2 sum alpha I, sum alpha I) becomes one term.
    std::vector<std::vector<std::pair<int32_t, double>>> rawA, rawB;
    auto canon_sum = [&](std::vector<std::pair<int32_t, double>>& v) {
      std::map<int32_t, double> acc;
      for (auto& e : v) acc[canon[e.first]] += e.second;
      v.clear();
      for (auto& e : acc)
        if (e.second != 0.0) v.push_back(e);
    };
    auto merge_side = [&](bool onB) {   // merge terms whose (onB ? B : A) side is one identical matrix
      std::vector<std::vector<std::pair<int32_t, double>>> nA, nB;
      std::map<int32_t, size_t> at;
      for (size_t q = 0; q < rawA.size(); ++q) {
        auto& key = onB ? rawB[q] : rawA[q];
        auto& other = onB ? rawA[q] : rawB[q];
        if (key.size() == 1) {
          const double wk = key[0].second;
          for (auto& e : other) e.second *= wk;
          key[0].second = 1.0;
          auto f = at.find(key[0].first);
          if (f != at.end()) {
            auto& o = onB ? nA[f->second] : nB[f->second];
            o.insert(o.end(), other.begin(), other.end());
            canon_sum(o);
            continue;
          }
          at[key[0].first] = nA.size();
        }
        nA.push_back(rawA[q]);
        nB.push_back(rawB[q]);
      }
      rawA.swap(nA);
      rawB.swap(nB);
    };
    auto merge_terms = [&]() {
      for (size_t q = 0; q < rawA.size(); ++q) {
        canon_sum(rawA[q]);
        canon_sum(rawB[q]);
      }
      for (size_t q = rawA.size(); q-- > 0;)   // drop terms that cancelled
        if (rawA[q].empty() || rawB[q].empty()) {
          rawA.erase(rawA.begin() + q);
          rawB.erase(rawB.begin() + q);
        }
      merge_side(true);
      merge_side(false);
      for (size_t q = rawA.size(); q-- > 0;)
        if (rawA[q].empty() || rawB[q].empty()) {
          rawA.erase(rawA.begin() + q);
          rawB.erase(rawB.begin() + q);
        }
    };
    for (int64_t m = 0; m < c.M; ++m) {
      const int32_t* gm = &c.WM[m * l];
      for (int64_t h = 0; h < c.L0; ++h) {
        const int32_t first = (int32_t)c.Hh.size();
        rawA.clear();
        rawB.clear();
        for (int32_t i = 0; i < gi->nterms; ++i) {
          const int64_t na = (int64_t)Wa_i[i].size() / l, nbm = (int64_t)Wb_i[i].size() / l;
          const bool byA = na <= nbm;   // one term per lambda (B summed) or per mu (A summed)
          for (int64_t u = 0; u < (byA ? na : nbm); ++u) {
            std::vector<std::pair<int32_t, double>> sum;
            for (int64_t v = 0; v < (byA ? nbm : na); ++v) {
              const int64_t lam = byA ? u : v, mu = byA ? v : u;
              for (int64_t x = 0; x < l; ++x)
                tmp[x] = gm[x] - c.Wp[h * l + x] - Wa_i[i][lam * l + x] - Wb_i[i][mu * l + x];
              const int64_t wv = multinomial(g.d2, tmp.data(), l);
              if (wv) sum.push_back({(int32_t)((byA ? c.gp_boff[i] + mu : c.gp_aoff[i] + lam)), (double)wv});
            }
            if (sum.empty()) continue;
            std::vector<std::pair<int32_t, double>> one{{(int32_t)(byA ? c.gp_aoff[i] + u : c.gp_boff[i] + u), 1.0}};
            rawA.push_back(byA ? one : sum);
            rawB.push_back(byA ? sum : one);
          }
        }
        merge_terms();
        for (size_t q = 0; q < rawA.size(); ++q) {
          tA.push_back(rawA[q]);
          tB.push_back(rawB[q]);
          c.Hh.push_back((int32_t)h);
          c.Hm.push_back((int32_t)m);
        }
        const int32_t cnt = (int32_t)c.Hh.size() - first;
        if (cnt) {
          c.Hidx[h * c.M + m] = first;
          c.Hcnt[h * c.M + m] = cnt;
        }
      }
    }
  }
  for (int64_t m = 0; m < c.M && !c.gen; ++m) {
    const int32_t* gm = &c.WM[m * l];
    for (int64_t h = 0; h < c.L0; ++h) {
      bool nz = false;
      for (int64_t a = 0; a < c.nA; ++a) {
        for (int64_t i = 0; i < l; ++i) tmp[i] = gm[i] - c.Wp[h * l + i] - c.Wa[a * l + i];
        int64_t v = multinomial(g.d2, tmp.data(), l);
        w[a] = (double)v;
        if (v) nz = true;
      }
      if (!nz) continue;
      c.Hidx[h * c.M + m] = (int32_t)c.Hh.size();
      c.Hcnt[h * c.M + m] = 1;
      c.Hh.push_back((int32_t)h);
      c.Hm.push_back((int32_t)m);
      c.Hw.insert(c.Hw.end(), w.begin(), w.end());
    }
  }
  const int64_t nnzH = (int64_t)c.Hh.size();

  // ---- block partition (SHARD_BLOCKS): contiguous cost-balanced ranges [b0, b1) -------------------
  // A block's share of the Schur work is sum over its active (h, h') pairs of n^4 per raw term:
  // nu_j^2 for a P-block, 4 mu_m^2 for a Lyapunov block; ties go to the lower index.
  c.b0 = 0;
  c.b1 = c.nb;
  if (g.shard == POLYA_SHARD_BLOCKS) {
    std::vector<double> bc(c.nb + 1, 0.0);
    for (int64_t j = 0; j < c.L; ++j) {
      int64_t nu = 0;
      for (int64_t h = 0; h < c.L0; ++h) nu += c.beta[h * c.L + j] != 0;
      bc[j + 1] = bc[j] + (double)(nu * nu);
    }
    for (int64_t m = 0; m < c.M; ++m) {
      int64_t mu = 0;
      for (int64_t h = 0; h < c.L0; ++h) mu += c.Hcnt[h * c.M + m];
      bc[c.L + m + 1] = bc[c.L + m] + 4.0 * (double)(mu * mu);
    }
    auto at = [&](int64_t r) -> int64_t {
      if (r <= 0) return 0;
      if (r >= g.nranks) return c.nb;
      const double target = bc[c.nb] * (double)r / (double)g.nranks;
      return std::lower_bound(bc.begin(), bc.end(), target) - bc.begin();
    };
    c.b0 = at(g.rank);
    c.b1 = std::max(c.b0, at(g.rank + 1));
  }
  auto owned = [&](int64_t b) { return b >= c.b0 && b < c.b1; };

  // ---- pairs (h <= h'), their k-entries, work items, rank partition ---------------------------
  c.npairs = c.L0 * (c.L0 + 1) / 2;
  std::vector<int32_t> ph(c.npairs), ph2(c.npairs);
  std::vector<int64_t> pK(c.npairs), pKpad(c.npairs), pItems(c.npairs), pMu(c.npairs);
  {
    int64_t p = 0;
    for (int64_t h = 0; h < c.L0; ++h)
      for (int64_t h2 = h; h2 < c.L0; ++h2, ++p) {
        ph[p] = (int32_t)h;
        ph2[p] = (int32_t)h2;
        int64_t mu = 0, nu = 0;
        for (int64_t m = 0; m < c.M; ++m)
          if (owned(c.L + m)) mu += (int64_t)c.Hcnt[h * c.M + m] * c.Hcnt[h2 * c.M + m];  // (q, q') entries
        for (int64_t j = 0; j < c.L; ++j)
          if (owned(j) && c.beta[h * c.L + j] && c.beta[h2 * c.L + j]) ++nu;
        pMu[p] = mu;
        pK[p] = 4 * mu + nu;                        // K_pair = 4 mu_hh' + nu_hh' (algorithmic)
        pKpad[p] = std::max<int64_t>(kKStage, (pK[p] + kKStage - 1) / kKStage * kKStage);  // whole stages, >= 1
        pItems[p] = (h == h2) ? c.ncls * (c.ncls + 1) / 2 : c.ncls * c.ncls;
      }
  }
  c.pair_item_global.assign(c.npairs + 1, 0);
  std::vector<double> cost_prefix(c.npairs + 1, 0.0);
  double n4 = (double)c.nbas * c.nbas * c.nbas * c.nbas;
  c.useful_flops_total = 0;
  for (int64_t p = 0; p < c.npairs; ++p) {
    c.pair_item_global[p + 1] = add_chk(c.pair_item_global[p], pItems[p]);
    cost_prefix[p + 1] = cost_prefix[p] + (double)pItems[p] * (double)std::max<int64_t>(pKpad[p], 1);
    c.useful_flops_total += (ph[p] == ph2[p] ? 1.0 : 2.0) * n4 * (double)pK[p];
  }
  c.items_total = c.pair_item_global[c.npairs];
  auto item_at_cost = [&](double target) -> int64_t {
    if (target <= 0) return 0;
    if (target >= cost_prefix[c.npairs]) return c.items_total;
    int64_t p = std::upper_bound(cost_prefix.begin(), cost_prefix.end(), target) - cost_prefix.begin() - 1;
    double per = (double)std::max<int64_t>(pKpad[p], 1);
    int64_t within = (int64_t)std::ceil((target - cost_prefix[p]) / per);
    return std::min(c.pair_item_global[p] + within, c.pair_item_global[p + 1]);
  };
  const double total_cost = cost_prefix[c.npairs];
  c.item0 = item_at_cost(total_cost * g.rank / g.nranks);
  c.item1 = item_at_cost(total_cost * (g.rank + 1) / g.nranks);
  if (g.rank == g.nranks - 1) c.item1 = c.items_total;
  if (g.rank == 0) c.item0 = 0;
  if (g.shard == POLYA_SHARD_BLOCKS) {  // every rank assembles all entries of its partial sum
    c.item0 = 0;
    c.item1 = c.items_total;
  }
  c.pair0 = c.pair1 = 0;
  if (c.item1 > c.item0) {
    c.pair0 = std::upper_bound(c.pair_item_global.begin(), c.pair_item_global.end(), c.item0) -
              c.pair_item_global.begin() - 1;
    c.pair1 = std::upper_bound(c.pair_item_global.begin(), c.pair_item_global.end(), c.item1 - 1) -
              c.pair_item_global.begin();
  }
  // local pairs and the kernel's item numbering: a contiguous pair range with the global item
  // prefix (TILES, BLOCKS), or the pairs (h, h') with h = rank mod nranks numbered from 0 (CYCLIC)
  c.local_pairs.clear();
  c.local_item.clear();
  c.pair_local.assign(c.npairs, -1);
  if (g.shard == POLYA_SHARD_CYCLIC) {
    c.local_item.push_back(0);
    for (int64_t p = 0; p < c.npairs; ++p)
      if (ph[p] % g.nranks == g.rank) {
        c.pair_local[p] = (int32_t)c.local_pairs.size();
        c.local_pairs.push_back(p);
        c.local_item.push_back(c.local_item.back() + pItems[p]);
      }
    c.item0 = 0;
    c.item1 = c.local_item.back();
    c.pair0 = c.local_pairs.empty() ? 0 : c.local_pairs.front();
    c.pair1 = c.local_pairs.empty() ? 0 : c.local_pairs.back() + 1;
  } else {
    for (int64_t p = c.pair0; p < c.pair1; ++p) {
      c.pair_local[p] = (int32_t)c.local_pairs.size();
      c.local_pairs.push_back(p);
      c.local_item.push_back(c.pair_item_global[p]);
    }
    c.local_item.push_back(c.pair_item_global[c.pair1]);
  }
  c.useful_flops_rank = 0;
  for (size_t q = 0; q < c.local_pairs.size(); ++q) {
    const int64_t p = c.local_pairs[q];
    const int64_t lo = g.shard == POLYA_SHARD_CYCLIC ? c.local_item[q] : c.pair_item_global[p];
    const int64_t a = std::max(c.item0, lo), b = std::min(c.item1, lo + pItems[p]);
    c.useful_flops_rank += (ph[p] == ph2[p] ? 1.0 : 2.0) * n4 * pK[p] * (double)(b - a) / (double)pItems[p];
  }
  c.npairs_local = (int64_t)c.local_pairs.size();
  if (!device) return;  // polya_plan: host-side bookkeeping only

  // ---- arena layout --------------------------------------------------------------------------
  // Q, R: one per (local pair, Lyapunov block active for both rows)
  int64_t nQR = 0;
  for (int64_t p : c.local_pairs) nQR += pMu[p];
  c.nQR = nQR;
  int64_t id = 0;
  c.id_X = id; id += c.nb;
  c.id_W = id; id += c.nb;
  c.id_H = id; id += nnzH;
  c.id_U = id; id += nnzH;
  c.id_V = id; id += nnzH;
  c.id_Ut = id; id += nnzH;
  c.id_Vt = id; id += nnzH;
  c.id_Zero = id; id += 1;
  c.id_Xb = id; id += c.nnz_beta;
  c.id_Wb = id; id += c.nnz_beta;
  const int64_t qr_per = c.gen ? 4 : 1;   // generalised: L1..L4 and R1..R4 per (pair, m, q, q')
  c.id_Q = id; id += qr_per * nQR;
  c.id_R = id; id += qr_per * nQR;
  c.id_Xt = id; id += c.nb;
  c.id_T = id; id += nnzH;
  c.id_Vy = id; id += c.L0;
  c.id_S = id; id += c.M;
  if (c.gen) {
    c.id_B = id; id += nnzH;      // B_t
    c.id_Abar = id; id += nnzH;   // A_t^T
    c.id_XA = id; id += nnzH;     // Xs A_t (adjoint)
    c.id_VB = id; id += nnzH;     // V_h(y) B_t (apply)
  }
  c.nmats = id;
  if (c.nmats > INT32_MAX) throw Fail{POLYA_EOVERFLOW, "too many arena matrices"};
  c.arena = dalloc<double>(mul_chk(c.nmats, c.mstride));
  CU(cudaMemset(c.arena, 0, (size_t)c.nmats * c.mstride * sizeof(double)));

  // ---- pre-scaled P-block copies beta_hj X_j, beta_hj W_j (kernel scale_copy) -----------------
  {
    std::vector<int32_t> dst, src;
    std::vector<double> w;
    for (size_t e = 0; e < be_src.size(); ++e) {
      dst.push_back((int32_t)(c.id_Xb + e)); src.push_back((int32_t)(c.id_X + be_src[e])); w.push_back(be_w[e]);
      dst.push_back((int32_t)(c.id_Wb + e)); src.push_back((int32_t)(c.id_W + be_src[e])); w.push_back(be_w[e]);
    }
    c.n_sc = (int64_t)dst.size();
    c.d_sc_dst = dupload(dst);
    c.d_sc_src = dupload(src);
    c.d_sc_w = dupload(w);
  }

  // ---- batched GEMM descriptors ---------------------------------------------------------------
  {
    std::vector<GemmItem> it;
    std::vector<GemmTerm> tm;
    // U_t = H_t X_{L+m}, V_t = H_t W_{L+m}, and their transposes X H_t^T, W H_t^T   (a7)
    for (int64_t t = 0; t < nnzH; ++t) {
      int32_t b = (int32_t)(c.L + c.Hm[t]);
      if (!owned(b)) continue;   // SHARD_BLOCKS: only this rank's Lyapunov blocks enter its partial G
      if (c.gen) {   // U = B X, V = B W, Ut = A^T X, Vt = A^T W
        const int32_t ids[4][2] = {{(int32_t)(c.id_B + t), (int32_t)(c.id_X + b)}, {(int32_t)(c.id_B + t), (int32_t)(c.id_W + b)},
                                   {(int32_t)(c.id_Abar + t), (int32_t)(c.id_X + b)}, {(int32_t)(c.id_Abar + t), (int32_t)(c.id_W + b)}};
        const int64_t dst[4] = {c.id_U, c.id_V, c.id_Ut, c.id_Vt};
        for (int k = 0; k < 4; ++k) {
          it.push_back({(int32_t)(dst[k] + t), (int32_t)tm.size(), (int32_t)tm.size() + 1, -1});
          tm.push_back({ids[k][0], ids[k][1], 0, 0, 1.0});
        }
        continue;
      }
      // X, W symmetric (polya_schur's contract), so X H^T = U^T and W H^T = V^T: stored by the same items
      it.push_back({(int32_t)(c.id_U + t), (int32_t)tm.size(), (int32_t)tm.size() + 1, (int32_t)(c.id_Ut + t)});
      tm.push_back({(int32_t)(c.id_H + t), (int32_t)(c.id_X + b), 0, 0, 1.0});
      it.push_back({(int32_t)(c.id_V + t), (int32_t)tm.size(), (int32_t)tm.size() + 1, (int32_t)(c.id_Vt + t)});
      tm.push_back({(int32_t)(c.id_H + t), (int32_t)(c.id_W + b), 0, 0, 1.0});
    }
    c.n_items_UV = (int64_t)it.size();
    c.d_items_UV = dupload(it);
    c.d_terms_UV = dupload(tm);
    c.rg = !c.gen && c.np <= 128;
    if (c.rg) {   // K3b groups: U_t, V_t of one block m share X_m, W_m (U^T, V^T by transposed stores)
      std::vector<std::vector<int32_t>> per_m((size_t)c.M);
      for (int64_t t = 0; t < nnzH; ++t)
        if (owned((int32_t)(c.L + c.Hm[t]))) per_m[(size_t)c.Hm[t]].push_back((int32_t)t);
      std::vector<RgGroup> grp;
      std::vector<RgEnt> ent;
      for (int64_t m = 0; m < c.M; ++m) {
        if (per_m[(size_t)m].empty()) continue;
        for (int w = 0; w < 2; ++w) {
          const int32_t e0 = (int32_t)ent.size();
          for (int32_t t : per_m[(size_t)m])
            ent.push_back({(int32_t)(c.id_H + t), (int32_t)((w ? c.id_V : c.id_U) + t), (int32_t)((w ? c.id_Vt : c.id_Ut) + t), 0});
          grp.push_back({(int32_t)((w ? c.id_W : c.id_X) + c.L + m), 0, e0, (int32_t)ent.size()});
        }
      }
      rg_upload(c, 0, grp, ent);
    }
    // adjoint: T_t = H_t Xt_{L+m}; generalised T_t = B_t (Xt_{L+m} A_t) (two passes)
    it.clear(); tm.clear();
    if (c.gen) {
      for (int64_t t = 0; t < nnzH; ++t) {
        it.push_back({(int32_t)(c.id_XA + t), (int32_t)tm.size(), (int32_t)tm.size() + 1, -1});
        tm.push_back({(int32_t)(c.id_Xt + c.L + c.Hm[t]), (int32_t)(c.id_Abar + t), 1, 0, 1.0});
      }
      c.n_items_T0 = (int64_t)it.size();
      c.d_items_T0 = dupload(it);
      c.d_terms_T0 = dupload(tm);
      it.clear(); tm.clear();
    }
    for (int64_t t = 0; t < nnzH; ++t) {
      it.push_back({(int32_t)(c.id_T + t), (int32_t)tm.size(), (int32_t)tm.size() + 1, -1});
      if (c.gen)
        tm.push_back({(int32_t)(c.id_B + t), (int32_t)(c.id_XA + t), 0, 0, 1.0});
      else
        tm.push_back({(int32_t)(c.id_H + t), (int32_t)(c.id_Xt + c.L + c.Hm[t]), 0, 0, 1.0});
    }
    c.n_items_T = (int64_t)it.size();
    c.d_items_T = dupload(it);
    c.d_terms_T = dupload(tm);
    if (c.rg) {   // K3b groups of the adjoint: the T_t of one block m share sym(X_m)
      std::vector<std::vector<int32_t>> per_m((size_t)c.M);
      for (int64_t t = 0; t < nnzH; ++t) per_m[(size_t)c.Hm[t]].push_back((int32_t)t);
      std::vector<RgGroup> grp;
      std::vector<RgEnt> ent;
      for (int64_t m = 0; m < c.M; ++m) {
        if (per_m[(size_t)m].empty()) continue;
        const int32_t e0 = (int32_t)ent.size();
        for (int32_t t : per_m[(size_t)m]) ent.push_back({(int32_t)(c.id_H + t), (int32_t)(c.id_T + t), -1, 0});
        grp.push_back({(int32_t)(c.id_Xt + c.L + m), 0, e0, (int32_t)ent.size()});
      }
      rg_upload(c, 2, grp, ent);
    }
    // apply: S_m = sum_h V_h(y) H_{h,m}; generalised S_m = sum_t A_t (V_h(y) B_t) (two passes)
    it.clear(); tm.clear();
    if (c.gen) {
      for (int64_t t = 0; t < nnzH; ++t) {
        it.push_back({(int32_t)(c.id_VB + t), (int32_t)tm.size(), (int32_t)tm.size() + 1, -1});
        tm.push_back({(int32_t)(c.id_Vy + c.Hh[t]), (int32_t)(c.id_B + t), 0, 0, 1.0});
      }
      c.n_items_S0 = (int64_t)it.size();
      c.d_items_S0 = dupload(it);
      c.d_terms_S0 = dupload(tm);
      it.clear(); tm.clear();
    }
    for (int64_t m = 0; m < c.M; ++m) {
      int32_t b0 = (int32_t)tm.size();
      for (int64_t h = 0; h < c.L0; ++h) {
        int32_t t = c.Hidx[h * c.M + m];
        if (t < 0) continue;
        if (c.gen) {
          for (int32_t q = t; q < t + c.Hcnt[h * c.M + m]; ++q)
            tm.push_back({(int32_t)(c.id_H + q), (int32_t)(c.id_VB + q), 0, 0, 1.0});
        } else {
          tm.push_back({(int32_t)(c.id_Vy + h), (int32_t)(c.id_H + t), 0, 0, 1.0});
        }
      }
      it.push_back({(int32_t)(c.id_S + m), b0, (int32_t)tm.size(), -1});
    }
    c.n_items_S = (int64_t)it.size();
    c.d_items_S = dupload(it);
    c.d_terms_S = dupload(tm);
  }

  // ---- Schur tables for this rank's pairs ------------------------------------------------------
  {
    std::vector<int32_t> qh, qh2, kL, kR;
    std::vector<int64_t> kbeg, pitem;
    std::vector<std::vector<RgEnt>> rgQ(c.rg ? (size_t)nnzH : 0), rgR(c.rg ? (size_t)nnzH : 0);   // K3b, by H operand
    std::vector<GemmItem> it;
    std::vector<GemmTerm> tm;
    int64_t q = 0;
    kbeg.push_back(0);
    pitem.push_back(c.local_item.empty() ? 0 : c.local_item[0]);
    for (size_t lp = 0; lp < c.local_pairs.size(); ++lp) {
      const int64_t p = c.local_pairs[lp];
      const int64_t h = ph[p], h2 = ph2[p];
      qh.push_back((int32_t)h);
      qh2.push_back((int32_t)h2);
      for (int64_t m = 0; m < c.M; ++m) {
        int32_t th = c.Hidx[h * c.M + m], th2 = c.Hidx[h2 * c.M + m];
        if (th < 0 || th2 < 0 || !owned(c.L + m)) continue;
        const int32_t b = (int32_t)(c.L + m);
        if (c.gen) {
          // F = -sum_q (A_q E B_q + B_q^T E A_q^T): per (q, q') the four (L, R) of tr(E_k L E_l R) are
          // (B X A', B' W A), (B X B'^T, A'^T W A), (A^T X A', B' W B^T), (A^T X B'^T, A'^T W B^T)
          // (reading R18; (H^T, I) gives back the four terms below)
          for (int32_t q1 = th; q1 < th + c.Hcnt[h * c.M + m]; ++q1)
            for (int32_t q2 = th2; q2 < th2 + c.Hcnt[h2 * c.M + m]; ++q2) {
              const int32_t Ab1 = (int32_t)(c.id_Abar + q1), Ab2 = (int32_t)(c.id_Abar + q2);
              const int32_t B1 = (int32_t)(c.id_B + q1), B2 = (int32_t)(c.id_B + q2);
              const int32_t spec[4][4] = {{(int32_t)(c.id_U + q1), Ab2, (int32_t)(c.id_V + q2), Ab1},
                                          {(int32_t)(c.id_U + q1), B2, (int32_t)(c.id_Vt + q2), Ab1},
                                          {(int32_t)(c.id_Ut + q1), Ab2, (int32_t)(c.id_V + q2), B1},
                                          {(int32_t)(c.id_Ut + q1), B2, (int32_t)(c.id_Vt + q2), B1}};
              for (int k = 0; k < 4; ++k) {
                const int32_t idL = (int32_t)(c.id_Q + 4 * q + k), idR = (int32_t)(c.id_R + 4 * q + k);
                it.push_back({idL, (int32_t)tm.size(), (int32_t)tm.size() + 1, -1});
                tm.push_back({spec[k][0], spec[k][1], 1, 0, 1.0});
                it.push_back({idR, (int32_t)tm.size(), (int32_t)tm.size() + 1, -1});
                tm.push_back({spec[k][2], spec[k][3], 1, 0, 1.0});
                kL.push_back(idL); kR.push_back(idR);
              }
              ++q;
            }
          continue;
        }
        const int32_t idQ = (int32_t)(c.id_Q + q), idR = (int32_t)(c.id_R + q);
        // Q_{hh'} = U_h H_{h'}^T,  R_{h'h} = V_{h'} H_h^T
        if (c.rg) {
          rgQ[(size_t)th2].push_back({(int32_t)(c.id_U + th), idQ, -1, 0});
          rgR[(size_t)th].push_back({(int32_t)(c.id_V + th2), idR, -1, 0});
        }
        it.push_back({idQ, (int32_t)tm.size(), (int32_t)tm.size() + 1, -1});
        tm.push_back({(int32_t)(c.id_U + th), (int32_t)(c.id_H + th2), 1, 0, 1.0});
        it.push_back({idR, (int32_t)tm.size(), (int32_t)tm.size() + 1, -1});
        tm.push_back({(int32_t)(c.id_V + th2), (int32_t)(c.id_H + th), 1, 0, 1.0});
        ++q;
        // T1 = U_{h'}^T[b1,c1] V_h^T[d1,a1]; T2 = X[b1,c1] R_{h'h}[d1,a1];
        // T3 = Q_{hh'}[b1,c1] W[d1,a1];     T4 = U_h[b1,c1] V_{h'}[d1,a1]   (O7)
        kL.push_back((int32_t)(c.id_Ut + th2)); kR.push_back((int32_t)(c.id_Vt + th));
        kL.push_back((int32_t)(c.id_X + b));   kR.push_back(idR);                    
        kL.push_back(idQ);                     kR.push_back((int32_t)(c.id_W + b));  
        kL.push_back((int32_t)(c.id_U + th));  kR.push_back((int32_t)(c.id_V + th2));
      }
      for (int64_t j = 0; j < c.L; ++j) {
        int64_t b1 = c.beta[h * c.L + j], b2 = c.beta[h2 * c.L + j];
        if (!b1 || !b2 || !owned(j)) continue;
        // P-block term beta_hj beta_h'j X_j (x) W_j as (beta_hj X_j) (x) (beta_h'j W_j)
        kL.push_back((int32_t)(c.id_Xb + bidx[h * c.L + j])); kR.push_back((int32_t)(c.id_Wb + bidx[h2 * c.L + j]));
      }
      // zero terms up to a whole stage; a pair with no common block still gets one (all-zero)
      // stage so that every work item flows through the K4 pipeline
      while ((int64_t)(kL.size() - kbeg.back()) % kKStage || (int64_t)kL.size() == kbeg.back()) {
        kL.push_back((int32_t)c.id_Zero); kR.push_back((int32_t)c.id_Zero);
      }
      kbeg.push_back((int64_t)kL.size());
      pitem.push_back(c.local_item[lp + 1]);
    }
    c.nk_local = (int64_t)kL.size();
    if (c.rg) {   // K3b groups: the Q (R) of one H_{t} operand (one h, one block m) share it
      std::vector<RgGroup> grp;
      std::vector<RgEnt> ent;
      for (int64_t t = 0; t < nnzH; ++t)
        for (auto* lst : {&rgQ[(size_t)t], &rgR[(size_t)t]}) {
          if (lst->empty()) continue;
          const int32_t e0 = (int32_t)ent.size();
          ent.insert(ent.end(), lst->begin(), lst->end());
          grp.push_back({(int32_t)(c.id_H + t), 1, e0, (int32_t)ent.size()});
        }
      rg_upload(c, 1, grp, ent);
    }
    c.n_items_QR = (int64_t)it.size();
    c.d_items_QR = dupload(it);
    c.d_terms_QR = dupload(tm);
    c.st.pair_h = dupload(qh);
    c.st.pair_h2 = dupload(qh2);
    c.st.pair_kbeg = dupload(kbeg);
    c.st.pair_item = dupload(pitem);
    {  // schedule of the whole share: local pairs by decreasing padded k-list (stable), their items in order
      std::vector<int32_t> order;
      for (int64_t q = 0; q < c.npairs_local; ++q)
        if (std::min(c.item1, c.local_item[q + 1]) > std::max(c.item0, c.local_item[q])) order.push_back((int32_t)q);
      std::stable_sort(order.begin(), order.end(),
                       [&](int32_t a, int32_t b) { return kbeg[a + 1] - kbeg[a] > kbeg[b + 1] - kbeg[b]; });
      std::vector<int64_t> lo, pre{0};
      for (int32_t q : order) {
        const int64_t a = std::max(c.item0, c.local_item[q]), b = std::min(c.item1, c.local_item[q + 1]);
        lo.push_back(a);
        pre.push_back(pre.back() + (b - a));
      }
      c.st.nsched = (int64_t)order.size();
      if (c.st.nsched > 0) {
        c.st.sched_pl = dupload(order);
        c.st.sched_lo = dupload(lo);
        c.st.sched_prefix = dupload(pre);
      }
    }
    {
      std::vector<int2> kd(kL.size());
      for (size_t i = 0; i < kL.size(); ++i) kd[i] = make_int2(kL[i], kR[i]);
      c.st.kdesc = dupload(kd);
    }
    std::vector<int32_t> ca, cb;   // chunk classes {i <= j}, row-major
    for (int64_t i = 0; i < c.r; ++i)
      for (int64_t j = i; j < c.r; ++j) { ca.push_back((int32_t)i); cb.push_back((int32_t)j); }
    c.st.cls_a = dupload(ca);
    c.st.cls_b = dupload(cb);
    c.st.counter = dalloc<unsigned long long>(1);
  }

  // ---- apply / adjoint tables -------------------------------------------------------------------
  {
    std::vector<int32_t> bbeg{0}, bh, hbeg{0}, hj, lbeg{0}, lt, lm;
    std::vector<double> bw, hw;
    for (int64_t j = 0; j < c.L; ++j) {
      for (int64_t h = 0; h < c.L0; ++h)
        if (c.beta[h * c.L + j]) { bh.push_back((int32_t)h); bw.push_back((double)c.beta[h * c.L + j]); }
      bbeg.push_back((int32_t)bh.size());
    }
    for (int64_t h = 0; h < c.L0; ++h) {
      for (int64_t j = 0; j < c.L; ++j)
        if (c.beta[h * c.L + j]) { hj.push_back((int32_t)j); hw.push_back((double)c.beta[h * c.L + j]); }
      hbeg.push_back((int32_t)hj.size());
      for (int64_t m = 0; m < c.M; ++m)
        for (int32_t t = c.Hidx[h * c.M + m]; t >= 0 && t < c.Hidx[h * c.M + m] + c.Hcnt[h * c.M + m]; ++t) {
          lt.push_back(t);
          lm.push_back((int32_t)m);
        }
      lbeg.push_back((int32_t)lt.size());
    }
    c.d_bP_beg = dupload(bbeg); c.d_bP_h = dupload(bh); c.d_bP_w = dupload(bw);
    c.d_hP_beg = dupload(hbeg); c.d_hP_j = dupload(hj); c.d_hP_w = dupload(hw);
    c.d_hL_beg = dupload(lbeg); c.d_hL_t = dupload(lt); c.d_hL_m = dupload(lm);
  }

  // ---- H on the device (kernel K1) ----------------------------------------------------------------
  if (c.gen) {   // A_t, A_t^T, B_t as weighted coefficient sums (k_wsum)
    const int64_t nn = c.n * c.n;
    std::vector<double> coef(coefN);   // the padded N x N coefficients of the terms, then R's
    std::vector<WsumItem> wi;
    std::vector<WsumTerm> wt;
    auto add = [&](int64_t dst, const std::vector<std::pair<int32_t, double>>& sum, int trans) {
      wi.push_back({(int32_t)dst, (int32_t)wt.size(), (int32_t)(wt.size() + sum.size()), trans});
      for (auto& p : sum) wt.push_back({p.first, 0, p.second});
    };
    for (int64_t t = 0; t < nnzH; ++t) {
      add(c.id_H + t, tA[t], 0);
      add(c.id_Abar + t, tA[t], 1);
      add(c.id_B + t, tB[t], 0);
    }
    c.n_ws = (int64_t)wi.size();
    c.d_ws_items = dupload(wi);
    c.d_ws_terms = dupload(wt);
    if (c.r_cnt) coef.insert(coef.end(), gi->R, gi->R + c.r_cnt * nn);
    // C_{L+m} = sum_rho multinomial(d2; gamma_m - rho) R_rho (exact integer weights; host, once)
    if (c.r_cnt) {
      std::vector<int32_t> Wr;
      enumerate(l, (int64_t)g.dp + g.da, Wr);
      std::vector<double> CL((size_t)c.M * nn, 0.0);
      for (int64_t m = 0; m < c.M; ++m)
        for (int64_t r = 0; r < c.r_cnt; ++r) {
          for (int64_t x = 0; x < l; ++x) tmp[x] = c.WM[m * l + x] - Wr[r * l + x];
          const int64_t wv = multinomial(g.d2, tmp.data(), l);
          if (!wv) continue;
          for (int64_t e = 0; e < nn; ++e) CL[m * nn + e] += (double)wv * gi->R[r * nn + e];
        }
      c.d_CL = dupload(CL);
    }
    c.d_coef = dupload(coef);
    CU(launch_wsum(c, 0));
    CU(cudaDeviceSynchronize());
    return;
  }
  c.dA = dalloc<double>(mul_chk(c.nA, mul_chk(c.n, c.n)));
  CU(cudaMemcpy(c.dA, A_host, (size_t)c.nA * c.n * c.n * sizeof(double), cudaMemcpyHostToDevice));
  c.dHw = dupload(c.Hw);
  CU(launch_setup_H(c, 0));
  CU(cudaDeviceSynchronize());
}

void free_ctx(Ctx& c) {
  for (int ph = 0; ph < Ctx::kRgPhases; ++ph) {
    if (c.d_rg_grp[ph]) cudaFree(c.d_rg_grp[ph]);
    if (c.d_rg_ent[ph]) cudaFree(c.d_rg_ent[ph]);
    if (c.d_rg_tile[ph]) cudaFree(c.d_rg_tile[ph]);
  }
  void* ps[] = {c.arena, c.dA, c.dHw, c.d_items_UV, c.d_terms_UV, c.d_items_QR, c.d_terms_QR,
                c.d_items_T, c.d_terms_T, c.d_sc_dst, c.d_sc_src, c.d_sc_w, c.d_items_S, c.d_terms_S, c.d_bP_beg, c.d_bP_h, c.d_bP_w,
                c.d_hP_beg, c.d_hP_j, c.d_hP_w, c.d_hL_beg, c.d_hL_t, c.d_hL_m, c.st.pair_h, c.st.pair_h2,
                c.st.pair_kbeg, c.st.pair_item, c.st.kdesc,
                c.st.cls_a, c.st.cls_b, c.st.counter, c.st.sched_pl, c.st.sched_lo, c.st.sched_prefix, c.d_coef, c.d_ws_items, c.d_ws_terms, c.d_items_T0,
                c.d_terms_T0, c.d_items_S0, c.d_terms_S0, c.d_CL};
  for (void* p : ps)
    if (p) cudaFree(p);
}

polya_status fail(polya_ctx* ctx, const Fail& f) {
  if (ctx) ctx->c.last_error = f.msg;
  return f.s;
}

}  // namespace

// ---- ABI ----------------------------------------------------------------------------------------

extern "C" polya_status polya_setup(const polya_config* cfg, const double* A_host, polya_ctx** out) {
  if (!out) return POLYA_EINVAL;
  *out = nullptr;
  if (!cfg || !A_host) return POLYA_EINVAL;
  const polya_config& g = *cfg;
  if (g.n < 1 || g.l < 1 || g.dp < 0 || g.da < 0 || g.d1 < 0 || g.d2 < 0 || !(g.delta > 0) || g.nranks < 1 ||
      g.rank < 0 || g.rank >= g.nranks || (g.shard < POLYA_SHARD_TILES || g.shard > POLYA_SHARD_CYCLIC))
    return POLYA_EINVAL;
  polya_ctx* ctx = new (std::nothrow) polya_ctx();
  if (!ctx) return POLYA_ENOMEM;
  ctx->c.cfg = g;
  try {
    if (cudaGetDevice(&ctx->c.device) != cudaSuccess) throw Fail{POLYA_ECUDA, "no CUDA device"};
    build(ctx->c, A_host);
  } catch (const Fail& f) {
    polya_status s = f.s;
    fprintf(stderr, "polya_setup: %s\n", f.msg.c_str());
    free_ctx(ctx->c);
    delete ctx;
    return s;
  } catch (const std::bad_alloc&) {
    free_ctx(ctx->c);
    delete ctx;
    return POLYA_ENOMEM;
  }
  *out = ctx;
  return POLYA_OK;
}

extern "C" polya_status polya_setup_general(const polya_config* cfg, int32_t nlmi, int32_t nterms,
                                           const int32_t* deg_a, const int32_t* deg_b, const double* At,
                                           const double* Bt, const double* R, polya_ctx** out) {
  if (!out) return POLYA_EINVAL;
  *out = nullptr;
  if (!cfg || nterms < 1 || !deg_a || !deg_b || !At || !Bt) return POLYA_EINVAL;
  const polya_config& g = *cfg;
  if (g.n < 1 || g.l < 1 || g.dp < 0 || g.da < 0 || g.d1 < 0 || g.d2 < 0 || !(g.delta > 0) || g.nranks < 1 ||
      g.rank < 0 || g.rank >= g.nranks || (g.shard < POLYA_SHARD_TILES || g.shard > POLYA_SHARD_CYCLIC))
    return POLYA_EINVAL;
  if (nlmi != 0 && nlmi < g.n) return POLYA_EINVAL;
  for (int32_t i = 0; i < nterms; ++i)   // every term homogeneous of the one total degree cfg->da (R18)
    if (deg_a[i] < 0 || deg_b[i] < 0 || deg_a[i] + deg_b[i] != g.da) return POLYA_EINVAL;
  polya_ctx* ctx = new (std::nothrow) polya_ctx();
  if (!ctx) return POLYA_ENOMEM;
  ctx->c.cfg = g;
  const GenInput gi{nterms, deg_a, deg_b, At, Bt, R, nlmi};
  try {
    if (cudaGetDevice(&ctx->c.device) != cudaSuccess) throw Fail{POLYA_ECUDA, "no CUDA device"};
    build(ctx->c, nullptr, true, &gi);
  } catch (const Fail& f) {
    polya_status s = f.s;
    fprintf(stderr, "polya_setup_general: %s\n", f.msg.c_str());
    free_ctx(ctx->c);
    delete ctx;
    return s;
  } catch (const std::bad_alloc&) {
    free_ctx(ctx->c);
    delete ctx;
    return POLYA_ENOMEM;
  }
  *out = ctx;
  return POLYA_OK;
}

static void fill_dims(const Ctx& c, polya_dims* o) {
  o->L0 = c.L0; o->L = c.L; o->M = c.M; o->nblocks = c.nb; o->Ntil = c.Ntil; o->K = c.K;
  o->nnz_beta = c.nnz_beta; o->nnz_H = (int64_t)c.Hh.size();
  o->npairs = c.npairs; o->pair0 = c.pair0; o->pair1 = c.pair1; o->item0 = c.item0; o->item1 = c.item1;
  o->useful_flops_schur = c.useful_flops_rank;
  o->tiles_bytes = c.npairs_local * c.Ntil * c.Ntil * (int64_t)sizeof(double);
  o->b0 = c.b0;
  o->b1 = c.b1;
  int64_t t = 0, groups = 0;
  combine_shape(c, &t, &groups);
  const bool blocks = c.cfg.shard == POLYA_SHARD_BLOCKS;
  o->reduce_count = blocks ? groups * t * c.Ntil * c.Ntil : 0;
  o->npairs_local = c.npairs_local;
  o->block_n = c.n;
  o->combine_tiles = blocks ? t : 0;
}

extern "C" polya_status polya_plan(const polya_config* cfg, polya_dims* out) {
  if (!cfg || !out) return POLYA_EINVAL;
  const polya_config& g = *cfg;
  if (g.n < 1 || g.l < 1 || g.dp < 0 || g.da < 0 || g.d1 < 0 || g.d2 < 0 || !(g.delta > 0) || g.nranks < 1 ||
      g.rank < 0 || g.rank >= g.nranks || (g.shard < POLYA_SHARD_TILES || g.shard > POLYA_SHARD_CYCLIC))
    return POLYA_EINVAL;
  try {
    Ctx c;
    c.cfg = g;
    build(c, nullptr, false);
    fill_dims(c, out);
  } catch (const Fail& f) {
    return f.s;
  } catch (const std::bad_alloc&) {
    return POLYA_ENOMEM;
  }
  return POLYA_OK;
}

// ---- homogenisation and simplex maps (set-up of non-homogeneous / non-simplex problems) ----------

extern "C" polya_status polya_homogenize(int32_t l, int32_t n, int32_t nterms, const int32_t* exps,
                                         const double* coeffs, int32_t* da_out, double* out) {
  if (l < 1 || n < 1 || nterms < 1 || !exps || !da_out || (out && !coeffs)) return POLYA_EINVAL;
  int32_t da = 0;
  for (int32_t t = 0; t < nterms; ++t) {
    int32_t d = 0;
    for (int32_t i = 0; i < l; ++i) {
      if (exps[(int64_t)t * l + i] < 0) return POLYA_EINVAL;
      d += exps[(int64_t)t * l + i];
    }
    da = std::max(da, d);
  }
  *da_out = da;
  if (!out) return POLYA_OK;   // size query
  try {
    std::vector<int32_t> W;
    enumerate(l, da, W);
    const int64_t cnt = (int64_t)W.size() / l, nn = (int64_t)n * n;
    std::fill(out, out + cnt * nn, 0.0);
    std::vector<int32_t> diff(l);
    for (int32_t t = 0; t < nterms; ++t) {
      int32_t d = 0;
      for (int32_t i = 0; i < l; ++i) d += exps[(int64_t)t * l + i];
      // (sum_j alpha_j)^{da - d} alpha^{e_t} = sum_gamma multinomial(da - d; gamma - e_t) alpha^gamma
      for (int64_t g = 0; g < cnt; ++g) {
        for (int32_t i = 0; i < l; ++i) diff[i] = W[g * l + i] - exps[(int64_t)t * l + i];
        const int64_t w = multinomial(da - d, diff.data(), l);
        if (!w) continue;
        for (int64_t e = 0; e < nn; ++e) out[g * nn + e] += (double)w * coeffs[(int64_t)t * nn + e];
      }
    }
  } catch (const Fail& f) {
    return f.s;
  }
  return POLYA_OK;
}

extern "C" polya_status polya_simplex_map(int32_t l, int32_t d, int32_t n, const double* scale, const double* shift,
                                          const double* A_in, double* A_out) {
  if (l < 1 || d < 0 || n < 1 || !scale || !shift || !A_in || !A_out) return POLYA_EINVAL;
  try {
    // exponent -> position in W_k, for k = 0..d
    std::vector<std::vector<int32_t>> W(d + 1);
    std::vector<std::map<std::vector<int32_t>, int64_t>> pos(d + 1);
    for (int32_t k = 0; k <= d; ++k) {
      enumerate(l, k, W[k]);
      for (int64_t q = 0; q < (int64_t)W[k].size() / l; ++q)
        pos[k][std::vector<int32_t>(W[k].begin() + q * l, W[k].begin() + (q + 1) * l)] = q;
    }
    const int64_t cnt = (int64_t)W[d].size() / l, nn = (int64_t)n * n;
    std::fill(A_out, A_out + cnt * nn, 0.0);
    for (int64_t q = 0; q < cnt; ++q) {
      // prod_i g_i(alpha)^{lambda_i}, g_i = scale_i alpha_i + shift_i sum_j alpha_j, by explicit
      // polynomial multiplication (dense coefficient vectors over W_k)
      std::vector<double> poly(1, 1.0);
      int32_t deg = 0;
      for (int32_t i = 0; i < l; ++i)
        for (int32_t r = 0; r < W[d][q * l + i]; ++r) {
          std::vector<double> next(W[deg + 1].size() / l, 0.0);
          std::vector<int32_t> e(l);
          for (int64_t u = 0; u < (int64_t)poly.size(); ++u) {
            if (poly[u] == 0.0) continue;
            for (int32_t j = 0; j < l; ++j) {
              const double cij = shift[i] + (j == i ? scale[i] : 0.0);
              if (cij == 0.0) continue;
              for (int32_t v = 0; v < l; ++v) e[v] = W[deg][u * l + v] + (v == j ? 1 : 0);
              next[pos[deg + 1][e]] += poly[u] * cij;
            }
          }
          poly.swap(next);
          ++deg;
        }
      for (int64_t g = 0; g < cnt; ++g)
        if (poly[g] != 0.0)
          for (int64_t e = 0; e < nn; ++e) A_out[g * nn + e] += poly[g] * A_in[q * nn + e];
    }
  } catch (const Fail& f) {
    return f.s;
  } catch (const std::bad_alloc&) {
    return POLYA_ENOMEM;
  }
  return POLYA_OK;
}

extern "C" polya_status polya_dims_get(const polya_ctx* ctx, polya_dims* o) {
  if (!ctx || !o) return POLYA_EINVAL;
  fill_dims(ctx->c, o);
  return POLYA_OK;
}

extern "C" polya_status polya_get_exponents(const polya_ctx* ctx, int which, int32_t* out) {
  if (!ctx || !out) return POLYA_EINVAL;
  const Ctx& c = ctx->c;
  const std::vector<int32_t>* v = which == 0 ? &c.Wp : which == 1 ? &c.WL : which == 2 ? &c.WM : which == 3 ? &c.Wa : nullptr;
  if (!v) return POLYA_EINVAL;
  std::memcpy(out, v->data(), v->size() * sizeof(int32_t));
  return POLYA_OK;
}

extern "C" polya_status polya_get_beta(const polya_ctx* ctx, int64_t* out) {
  if (!ctx || !out) return POLYA_EINVAL;
  std::memcpy(out, ctx->c.beta.data(), ctx->c.beta.size() * sizeof(int64_t));
  return POLYA_OK;
}

extern "C" polya_status polya_get_C(const polya_ctx* ctx, double* out) {
  if (!ctx || !out) return POLYA_EINVAL;
  std::memcpy(out, ctx->c.c.data(), ctx->c.c.size() * sizeof(double));
  return POLYA_OK;
}

extern "C" polya_status polya_get_H(const polya_ctx* ctx, double* out) {
  if (!ctx || !out) return POLYA_EINVAL;
  const Ctx& c = ctx->c;
  if (c.gen) {
    const_cast<polya_ctx*>(ctx)->c.last_error = "polya_get_H: no H table in the generalised form";
    return POLYA_EINVAL;
  }
  const int64_t n = c.n, nn = n * n;
  std::memset(out, 0, (size_t)c.L0 * c.M * nn * sizeof(double));
  std::vector<double> buf(c.mstride);
  for (size_t t = 0; t < c.Hh.size(); ++t) {
    cudaError_t e = cudaMemcpy(buf.data(), c.arena + (c.id_H + (int64_t)t) * c.mstride, c.mstride * sizeof(double),
                               cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) {
      const_cast<polya_ctx*>(ctx)->c.last_error = cudaGetErrorString(e);
      return POLYA_ECUDA;
    }
    double* dst = out + ((int64_t)c.Hh[t] * c.M + c.Hm[t]) * nn;
    for (int64_t i = 0; i < n; ++i)
      for (int64_t j = 0; j < n; ++j) dst[i * n + j] = buf[i * c.np + j];
  }
  return POLYA_OK;
}

extern "C" polya_status polya_apply(polya_ctx* ctx, const double* y, double* out, void* stream) {
  if (!ctx || !y || !out) return POLYA_EINVAL;
  Ctx& c = ctx->c;
  cudaStream_t s = (cudaStream_t)stream;
  try {
    CU(launch_vmap(c, y, s));
    CU(launch_gemm(c, c.d_items_S0, c.d_terms_S0, c.n_items_S0, s));   // generalised form only
    CU(launch_gemm(c, c.d_items_S, c.d_terms_S, c.n_items_S, s));
    CU(launch_apply_out(c, y, out, s));
  } catch (const Fail& f) {
    return fail(ctx, f);
  }
  return POLYA_OK;
}

extern "C" polya_status polya_adjoint(polya_ctx* ctx, const double* X, double* y, void* stream) {
  if (!ctx || !X || !y) return POLYA_EINVAL;
  Ctx& c = ctx->c;
  cudaStream_t s = (cudaStream_t)stream;
  try {
    CU(launch_pad_copy(c, X, c.id_Xt, c.nb, 1, s));
    CU(launch_gemm(c, c.d_items_T0, c.d_terms_T0, c.n_items_T0, s));   // generalised form only
    if (c.rg)
      CU(launch_rgemm(c, 2, s));
    else
      CU(launch_gemm(c, c.d_items_T, c.d_terms_T, c.n_items_T, s));
    CU(launch_adjoint_reduce(c, y, s));
  } catch (const Fail& f) {
    return fail(ctx, f);
  }
  return POLYA_OK;
}

extern "C" polya_status polya_schur_prepare(polya_ctx* ctx, const double* X, const double* Zinv, void* stream) {
  if (!ctx || !X || !Zinv) return POLYA_EINVAL;
  Ctx& c = ctx->c;
  cudaStream_t s = (cudaStream_t)stream;
  try {
    if (c.timing) CU(cudaEventRecord(c.ev[0], s));
    CU(launch_pad_copy(c, X, c.id_X, c.nb, 0, s));
    CU(launch_pad_copy(c, Zinv, c.id_W, c.nb, 0, s));
    CU(launch_scale_copy(c, s));
    if (c.rg) {
      CU(launch_rgemm(c, 0, s));
      CU(launch_rgemm(c, 1, s));
    } else {
      CU(launch_gemm(c, c.d_items_UV, c.d_terms_UV, c.n_items_UV, s));
      CU(launch_gemm(c, c.d_items_QR, c.d_terms_QR, c.n_items_QR, s));
    }
    if (c.timing) CU(cudaEventRecord(c.ev[1], s));
  } catch (const Fail& f) {
    return fail(ctx, f);
  }
  return POLYA_OK;
}

extern "C" polya_status polya_schur_assemble(polya_ctx* ctx, double* G, int layout, int64_t pair_begin,
                                             int64_t pair_end, void* stream) {
  if (!ctx || !G) return POLYA_EINVAL;
  if (layout != POLYA_G_FULL && layout != POLYA_G_PAIR_TILES) return POLYA_EINVAL;
  Ctx& c = ctx->c;
  if (pair_begin < 0 || pair_end > c.npairs_local || pair_begin > pair_end) return POLYA_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  try {
    int64_t i0 = c.item0, i1 = c.item1;
    if (c.npairs_local > 0) {
      i0 = std::max(c.item0, c.local_item[pair_begin]);
      i1 = std::min(c.item1, c.local_item[pair_end]);
    }
    CU(launch_schur(c, G, layout, i0, i1, s));
    if (c.timing) CU(cudaEventRecord(c.ev[2], s));
  } catch (const Fail& f) {
    return fail(ctx, f);
  }
  return POLYA_OK;
}

extern "C" polya_status polya_schur(polya_ctx* ctx, const double* X, const double* Zinv, double* G, int layout,
                                    void* stream) {
  if (!ctx || !X || !Zinv || !G) return POLYA_EINVAL;
  if (layout != POLYA_G_FULL && layout != POLYA_G_PAIR_TILES) return POLYA_EINVAL;
  polya_status st = polya_schur_prepare(ctx, X, Zinv, stream);
  if (st != POLYA_OK) return st;
  return polya_schur_assemble(ctx, G, layout, 0, ctx->c.npairs_local, stream);
}

extern "C" polya_status polya_set_timing(polya_ctx* ctx, int enable) {
  if (!ctx) return POLYA_EINVAL;
  Ctx& c = ctx->c;
  if (enable && !c.ev[0]) {
    for (auto& e : c.ev)
      if (cudaEventCreate(&e) != cudaSuccess) {
        c.last_error = "cudaEventCreate failed";
        return POLYA_ECUDA;
      }
  }
  c.timing = enable != 0;
  return POLYA_OK;
}

extern "C" polya_status polya_get_timing(polya_ctx* ctx, float* ms_pre, float* ms_assemble) {
  if (!ctx || !ms_pre || !ms_assemble) return POLYA_EINVAL;
  Ctx& c = ctx->c;
  if (!c.ev[0]) return POLYA_EINVAL;
  if (cudaEventSynchronize(c.ev[2]) != cudaSuccess || cudaEventElapsedTime(ms_pre, c.ev[0], c.ev[1]) != cudaSuccess ||
      cudaEventElapsedTime(ms_assemble, c.ev[1], c.ev[2]) != cudaSuccess) {
    c.last_error = "timing events not recorded";
    return POLYA_ECUDA;
  }
  return POLYA_OK;
}

extern "C" polya_status polya_get_combine_timing(polya_ctx* ctx, float* ms_exposed) {
  if (!ctx || !ms_exposed) return POLYA_EINVAL;
  Ctx& c = ctx->c;
  if (!c.ev[0]) return POLYA_EINVAL;
  if (cudaEventSynchronize(c.ev[3]) != cudaSuccess || cudaEventElapsedTime(ms_exposed, c.ev[2], c.ev[3]) != cudaSuccess) {
    c.last_error = "combine timing events not recorded (polya_schur_reduce with timing on)";
    return POLYA_ECUDA;
  }
  return POLYA_OK;
}

extern "C" polya_status polya_sync(polya_ctx* ctx) {
  if (!ctx) return POLYA_EINVAL;
  cudaError_t e = cudaDeviceSynchronize();
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) {
    ctx->c.last_error = cudaGetErrorString(e);
    return POLYA_ECUDA;
  }
  return POLYA_OK;
}

extern "C" const char* polya_strerror(polya_status s) {
  switch (s) {
    case POLYA_OK: return "ok";
    case POLYA_EINVAL: return "invalid argument";
    case POLYA_EOVERFLOW: return "integer overflow in problem size";
    case POLYA_ENOMEM: return "out of memory";
    case POLYA_ECUDA: return "CUDA error";
    case POLYA_ENCCL: return "NCCL error";
    case POLYA_ENOTPD: return "matrix not positive definite";
    case POLYA_ESTEP: return "no admissible step";
    case POLYA_EMAXIT: return "iteration limit";
    case POLYA_EDIVERGED: return "iterates diverged (infeasible LMI)";
  }
  return "unknown status";
}

extern "C" const char* polya_last_error(const polya_ctx* ctx) { return ctx ? ctx->c.last_error.c_str() : ""; }

extern "C" int64_t polya_launch_count(const polya_ctx* ctx) { return ctx ? ctx->c.launches : 0; }

void polya_ipm_free(polya::Ctx& c);  // ipm.cu
namespace polya { void nccl_free(Ctx& c); }  // combine.cpp

extern "C" void polya_destroy(polya_ctx* ctx) {
  if (!ctx) return;
  polya_ipm_free(ctx->c);
  combine_free(ctx->c);
  nccl_free(ctx->c);
  for (auto& e : ctx->c.ev)
    if (e) cudaEventDestroy(e);
  free_ctx(ctx->c);
  delete ctx;
}
