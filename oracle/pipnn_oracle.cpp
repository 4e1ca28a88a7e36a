// pipnn_oracle.cpp — CPU ORACLE for the PiPNN build (arxiv 2602.21247). TEST INFRASTRUCTURE ONLY.
//
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may load
// this library. It shares no code, header, table or constant generator with the CUDA path under
// paper_2602_21247_b200/csrc; the shared randomness is re-implemented here from docs/DETERMINISM.md.
//
// What it computes, in the paper's order and notation (PAPER.md = "P:", SPEC.md = "S:"):
//   * dissimilarity ||.,.||: squared L2 or MIPS -<x,y>, direct form, fp64 (int64-exact
//     for uint8). Float data in "bf16" mode is first rounded to bf16 (reading R19).
//   * Alg. 5 Randomized Ball Carving with fanout + merge of small groups    -> or_partition
//   * leaf k-NN pick, bidirected                                 -> or_leaf_pick
//   * Eq. 1 residual hash via sketches and Alg. 3 HashPrune, run both
//     as the streaming algorithm and as the Supp. G characterization     -> or_hashprune
//   * final RobustPrune, Alg. 2 and its lazy form               -> or_final_prune
//   * Alg. 4 end to end                                                     -> or_build
//   * evaluation harness: exact k-NN (Def. 1), Alg. 1 beam search, recall (Def. 2).
// Plain loops; OpenMP only across independent units (points, leaves, owners, queries).
// parity pinned: every function is exercised by tests/test_oracle_*.py against SPEC/PAPER examples,
// closed forms, brute force and invariants.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <utility>
#include <vector>
#ifdef _OPENMP
#include <omp.h>
#endif

namespace {

// ------------------------------------------------------------------ randomness (docs/DETERMINISM.md)
const uint64_t DOM_H = 0x48595045524C4E45ull;
const uint64_t DOM_PART = 0x5041525449544E31ull;
const uint64_t DOM_MERGE = 0x4D45524745535444ull;

uint64_t splitmix_out(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
uint64_t mix(uint64_t a, uint64_t b) { return splitmix_out(a ^ splitmix_out(b)); }

// ------------------------------------------------------------------ bf16 helpers
uint16_t bf16_rne(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  u += 0x7FFFu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}
float bf16_to_float(uint16_t b) {
  uint32_t u = (uint32_t)b << 16;
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}
// okey: makes the bf16 bit pattern order like its value
uint16_t okey(uint16_t b) { return (uint16_t)(b ^ ((b & 0x8000u) ? 0xFFFFu : 0x8000u)); }
// stored reservoir distance key: canonicalise -0, round to fp32, then to bf16 (R5)
uint16_t dist_okey(double D) {
  float f = (float)D;
  f = f + 0.0f;
  return okey(bf16_rne(f));
}

double now_s() {
  using namespace std::chrono;
  return duration<double>(steady_clock::now().time_since_epoch()).count();
}

}  // namespace

extern "C" {

typedef struct {
  const void* data;
  int64_t n;
  int32_t d;
  int32_t dtype;   // 0 = uint8, 1 = float32
  int32_t metric;  // 0 = squared L2, 1 = MIPS (-<x,y>)
  int32_t mode;    // float only: 0 = exact (fp32 values), 1 = bf16 (values rounded to bf16 first)
} or_points;

typedef struct {
  int32_t c_max, c_min, p_num, p_den, leader_cap;
  int32_t fanout[4];
  int32_t n_fanout, replicas;
  int32_t k, m, l_max, R, alpha_num, alpha_den, final_prune;
  uint64_t seed;
} or_params;

typedef struct {
  int64_t n_leaves, n_instances;
  int64_t* leaf_off;
  uint32_t* leaf_ids;
  int32_t k;
  uint32_t* nbr;  // [n_instances * k]
  double* dist;   // [n_instances * k]
  int32_t l_max;
  uint64_t* slots;  // [n * l_max]
  uint32_t* count;  // [n]
  int64_t n_streamed;
  int64_t* row_ptr;  // [n + 1]
  uint32_t* col_idx; // [row_ptr[n]]
  int32_t depth;
  int32_t check_failed;  // bit 1: streaming != characterization; bit 2: eager != lazy
  double t_partition, t_leaf, t_hashprune, t_final, t_total;
} or_result;

}  // extern "C"

namespace {

// ------------------------------------------------------------------ dataset view + dissimilarity
struct Data {
  int64_t n = 0;
  int d = 0;
  bool u8 = false, mips = false;
  const uint8_t* xu = nullptr;
  std::vector<float> xf;  // float coordinates after the mode's rounding

  Data(const or_points* p, bool force_exact = false) {
    n = p->n;
    d = p->d;
    u8 = (p->dtype == 0);
    mips = (p->metric == 1);
    if (u8) {
      xu = (const uint8_t*)p->data;
    } else {
      const float* s = (const float*)p->data;
      xf.assign(s, s + (size_t)n * d);
      if (p->mode == 1 && !force_exact)
        for (auto& v : xf) v = bf16_to_float(bf16_rne(v));
    }
  }
  // ||a,b|| for two dataset points (direct form)
  double dist(int64_t a, int64_t b) const {
    if (u8) {
      const uint8_t* pa = xu + (size_t)a * d;
      const uint8_t* pb = xu + (size_t)b * d;
      int64_t s = 0;
      for (int j = 0; j < d; ++j) {
        int64_t t = (int64_t)pa[j] - (int64_t)pb[j];
        s += t * t;
      }
      return (double)s;
    }
    const float* pa = xf.data() + (size_t)a * d;
    const float* pb = xf.data() + (size_t)b * d;
    double s = 0;
    if (mips) {
      for (int j = 0; j < d; ++j) s += (double)pa[j] * (double)pb[j];
      return -s;
    }
    for (int j = 0; j < d; ++j) {
      double t = (double)pa[j] - (double)pb[j];
      s += t * t;
    }
    return s;
  }
  // The dissimilarity RobustPrune's alpha test is applied to (reading R22, changed): the dataset's own
  // measure for L2; for MIPS the angular dissimilarity 1 - <a,b>/(||a|| ||b||) (cosine 0 when a norm is 0).
  // alpha >= 1 relaxes the prune only on non-negative values; on the signed -<a,b> the
  // same product tightens it and the final prune leaves out-degree ~1 (R22).
  double dprune(int64_t a, int64_t b) const {
    if (!mips) return dist(a, b);
    const double ab = -dist(a, b), aa = -dist(a, a), bb = -dist(b, b);
    if (aa <= 0.0 || bb <= 0.0) return 1.0;
    return 1.0 - ab / (std::sqrt(aa) * std::sqrt(bb));
  }
  // ||q,b|| for an external query vector q given in fp64
  double dist_q(const double* q, int64_t b) const {
    double s = 0;
    if (u8) {
      const uint8_t* pb = xu + (size_t)b * d;
      for (int j = 0; j < d; ++j) {
        double t = q[j] - (double)pb[j];
        s += t * t;
      }
      return s;
    }
    const float* pb = xf.data() + (size_t)b * d;
    if (mips) {
      for (int j = 0; j < d; ++j) s += q[j] * (double)pb[j];
      return -s;
    }
    for (int j = 0; j < d; ++j) {
      double t = q[j] - (double)pb[j];
      s += t * t;
    }
    return s;
  }
  double coord(int64_t i, int j) const { return u8 ? (double)xu[(size_t)i * d + j] : (double)xf[(size_t)i * d + j]; }
};

// ------------------------------------------------------------------ hyperplanes + sketches
std::vector<int8_t> make_hyperplanes(int m, int d, uint64_t seed) {
  std::vector<int8_t> H((size_t)m * d);
  const uint64_t sH = mix(seed, DOM_H);
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < d; ++j) {
      int v = 0;
      for (int t = 0; t < 4; ++t) {
        uint64_t u = mix(sH, 4ull * ((uint64_t)i * d + j) + t) >> 59;
        v += 2 * (int)u - 31;
      }
      H[(size_t)i * d + j] = (int8_t)v;
    }
  return H;
}

// Sketch table as fp64 values (exact integers for u8; fp32-rounded values for float).
std::vector<double> make_sketches(const Data& X, const int8_t* H, int m) {
  std::vector<double> S((size_t)X.n * m);
#pragma omp parallel for schedule(static)
  for (int64_t x = 0; x < X.n; ++x)
    for (int i = 0; i < m; ++i) {
      if (X.u8) {
        int64_t s = 0;
        for (int j = 0; j < X.d; ++j) s += (int64_t)H[(size_t)i * X.d + j] * (int64_t)X.xu[(size_t)x * X.d + j];
        S[(size_t)x * m + i] = (double)s;
      } else {
        double s = 0;
        for (int j = 0; j < X.d; ++j) s += (double)H[(size_t)i * X.d + j] * (double)X.xf[(size_t)x * X.d + j];
        S[(size_t)x * m + i] = (double)(float)s;
      }
    }
  return S;
}

// Eq. 1 via sketches: bit i = [S(v)_i - S(u)_i >= 0]
uint32_t residual_hash(const double* Su, const double* Sv, int m) {
  uint32_t h = 0;
  for (int i = 0; i < m; ++i)
    if (Sv[i] >= Su[i]) h |= (1u << i);
  return h;
}

// Merge of small sibling groups ("merge partitions randomly (never exceeding C_max)").
// Reading R15: Small = {0 < |g| < C_min} in (mix(K^DOM_MERGE, l), l) order are accumulated into bins that
// close once the SUM of member-group sizes reaches C_min; a leftover joins the first closed bin, else the
// smallest Big group (ties by key) whose size + leftover sum <= C_max, else stands alone. With
// 3*C_min < C_max no bin can exceed C_max. Unions dedupe ids (fanout > 1 makes siblings overlap).
struct MergePlan {
  std::vector<int64_t> big;                 // big groups, in leader order
  std::vector<std::vector<int64_t>> bins;   // each: small groups unioned into one leaf
  std::vector<int64_t> leftover;            // small groups absorbed by big group `absorb_big`
  int64_t absorb_big = -1;
};
MergePlan merge_plan(const std::vector<int64_t>& sizes, const std::vector<std::pair<uint64_t, uint32_t>>& keys,
                     int64_t c_min, int64_t c_max) {
  MergePlan mp;
  const int64_t l = (int64_t)sizes.size();
  std::vector<int64_t> small;
  for (int64_t j = 0; j < l; ++j) {
    if (sizes[j] == 0) continue;
    if (sizes[j] < c_min) small.push_back(j);
    else mp.big.push_back(j);
  }
  std::sort(small.begin(), small.end(), [&](int64_t a, int64_t b) { return keys[a] < keys[b]; });
  std::vector<int64_t> cur;
  int64_t cur_sum = 0;
  for (int64_t j : small) {
    cur.push_back(j);
    cur_sum += sizes[j];
    if (cur_sum >= c_min) {
      mp.bins.push_back(cur);
      cur.clear();
      cur_sum = 0;
    }
  }
  if (!cur.empty()) {
    if (!mp.bins.empty()) {
      mp.bins[0].insert(mp.bins[0].end(), cur.begin(), cur.end());
    } else {
      for (int64_t j : mp.big) {
        if (sizes[j] + cur_sum > c_max) continue;
        if (mp.absorb_big < 0 || sizes[j] < sizes[mp.absorb_big] ||
            (sizes[j] == sizes[mp.absorb_big] && keys[j] < keys[mp.absorb_big]))
          mp.absorb_big = j;
      }
      if (mp.absorb_big < 0) mp.bins.push_back(cur);
      else mp.leftover = cur;
    }
  }
  return mp;
}

// ------------------------------------------------------------------ Alg. 5: Randomized Ball Carving
struct Carver {
  const Data& X;
  const or_params& P;
  std::vector<std::vector<uint32_t>>& leaves;
  int max_depth = 0;

  Carver(const Data& X_, const or_params& P_, std::vector<std::vector<uint32_t>>& L) : X(X_), P(P_), leaves(L) {}

  void emit_chunks(const std::vector<uint32_t>& g) {  // degenerate-input guard
    const int64_t sz = (int64_t)g.size();
    const int64_t nc = (sz + P.c_max - 1) / P.c_max;
    for (int64_t c = 0; c < nc; ++c) {
      int64_t lo = c * sz / nc, hi = (c + 1) * sz / nc;
      leaves.emplace_back(g.begin() + lo, g.begin() + hi);
    }
  }

  static std::vector<uint32_t> set_union(const std::vector<const std::vector<uint32_t>*>& parts) {
    std::vector<uint32_t> u;
    for (auto* p : parts) u.insert(u.end(), p->begin(), p->end());
    std::sort(u.begin(), u.end());
    u.erase(std::unique(u.begin(), u.end()), u.end());
    return u;
  }

  // P: ascending ids, |P| arbitrary.
  void carve(const std::vector<uint32_t>& Pset, int depth, uint64_t K) {
    max_depth = std::max(max_depth, depth);
    const int64_t sz = (int64_t)Pset.size();
    if (sz <= P.c_max) {  // line 1: base case
      leaves.push_back(Pset);
      return;
    }
    // line 2: SampleLeaders(P, P_samp*|P|), capped
    int64_t l = ((int64_t)P.p_num * sz + P.p_den - 1) / P.p_den;
    l = std::max<int64_t>(l, 2);
    l = std::min<int64_t>(l, P.leader_cap);
    l = std::min<int64_t>(l, sz);
    std::vector<std::pair<uint64_t, uint32_t>> pri(sz);
    for (int64_t i = 0; i < sz; ++i) pri[i] = {mix(K, Pset[i]), Pset[i]};
    std::partial_sort(pri.begin(), pri.begin() + l, pri.end());
    std::vector<uint32_t> L(l);
    for (int64_t j = 0; j < l; ++j) L[j] = pri[j].second;
    std::sort(L.begin(), L.end());
    // line 3: local fanout, clamped to the number of leaders
    int f = depth < P.n_fanout ? P.fanout[depth] : 1;
    f = (int)std::min<int64_t>(f, l);
    // lines 5-9: each x joins its f nearest leaders by (D(x,l), l)
    std::vector<int32_t> assign((size_t)sz * f);
#pragma omp parallel for schedule(dynamic, 64) if (sz * l > 200000)
    for (int64_t i = 0; i < sz; ++i) {
      std::vector<std::pair<double, int32_t>> dl(l);
      for (int64_t j = 0; j < l; ++j) dl[j] = {X.dist(Pset[i], L[j]), (int32_t)j};
      std::partial_sort(dl.begin(), dl.begin() + f, dl.end());
      for (int t = 0; t < f; ++t) assign[(size_t)i * f + t] = dl[t].second;
    }
    std::vector<std::vector<uint32_t>> G(l);
    for (int64_t i = 0; i < sz; ++i)
      for (int t = 0; t < f; ++t) G[assign[(size_t)i * f + t]].push_back(Pset[i]);

    // line 10: Merge(B, C_min, C_max) — DESIGN.md reading R15 (sum-of-sizes rule)
    std::vector<int64_t> sizes(l);
    std::vector<std::pair<uint64_t, uint32_t>> mkeys(l);
    const uint64_t KM = K ^ DOM_MERGE;
    for (int64_t j = 0; j < l; ++j) {
      sizes[j] = (int64_t)G[j].size();
      mkeys[j] = {mix(KM, L[j]), L[j]};
    }
    MergePlan mp = merge_plan(sizes, mkeys, P.c_min, P.c_max);
    const std::vector<int64_t>& big = mp.big;
    const int64_t absorb_big = mp.absorb_big;
    const std::vector<int64_t>& cur = mp.leftover;
    const std::vector<std::vector<int64_t>>& bins = mp.bins;
    // lines 11-14: leaves and recursion (big groups in leader order, then bins)
    for (int64_t j : big) {
      if (j == absorb_big) {
        std::vector<const std::vector<uint32_t>*> parts{&G[j]};
        for (int64_t s : cur) parts.push_back(&G[s]);
        leaves.push_back(set_union(parts));
        continue;
      }
      const std::vector<uint32_t>& g = G[j];
      if ((int64_t)g.size() <= P.c_max) {
        leaves.push_back(g);
      } else if ((int64_t)g.size() == sz || depth + 1 >= 64) {
        emit_chunks(g);
      } else {
        carve(g, depth + 1, mix(K, (uint64_t)L[j] + 1));
      }
    }
    for (auto& b : bins) {
      std::vector<const std::vector<uint32_t>*> parts;
      for (int64_t s : b) parts.push_back(&G[s]);
      leaves.push_back(set_union(parts));
    }
  }
};

void run_partition(const Data& X, const or_params& P, std::vector<std::vector<uint32_t>>& leaves, int& depth) {
  Carver cv(X, P, leaves);
  std::vector<uint32_t> all(X.n);
  for (int64_t i = 0; i < X.n; ++i) all[i] = (uint32_t)i;
  for (int r = 0; r < P.replicas; ++r) cv.carve(all, 0, mix(mix(P.seed, DOM_PART), (uint64_t)r));
  depth = cv.max_depth;
}

// ------------------------------------------------------------------ leaf pick: bidirected k-NN
void run_leaf_pick(const Data& X, const int64_t* off, const uint32_t* ids, int64_t nl, int k, uint32_t* nbr,
                   double* dist) {
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t b = 0; b < nl; ++b) {
    const int64_t s = off[b + 1] - off[b];
    const uint32_t* leaf = ids + off[b];
    const int64_t cnt = std::min<int64_t>(k, s - 1);
    std::vector<std::pair<double, uint32_t>> row;
    for (int64_t i = 0; i < s; ++i) {
      row.clear();
      for (int64_t j = 0; j < s; ++j)
        if (j != i) row.push_back({X.dist(leaf[i], leaf[j]), leaf[j]});
      std::partial_sort(row.begin(), row.begin() + cnt, row.end());
      uint32_t* on = nbr + (size_t)(off[b] + i) * k;
      double* od = dist + (size_t)(off[b] + i) * k;
      for (int t = 0; t < k; ++t) {
        on[t] = t < cnt ? row[t].second : 0xFFFFFFFFu;
        od[t] = t < cnt ? row[t].first : INFINITY;
      }
    }
  }
}

// ------------------------------------------------------------------ Alg. 3 HashPrune
struct Slot {
  uint32_t hash;
  uint16_t ok;
  uint32_t id;
  uint64_t key() const { return ((uint64_t)ok << 32) | id; }  // (dist, id) total order
  uint64_t packed() const { return ((uint64_t)hash << 48) | ((uint64_t)ok << 32) | id; }
};

// Streaming Alg. 3: strict "<" on (bf16 dist, id) keys.
std::vector<Slot> hashprune_stream(const std::vector<Slot>& stream, int lmax) {
  std::vector<Slot> M;
  for (const Slot& c : stream) {
    int hit = -1;
    for (size_t i = 0; i < M.size(); ++i)
      if (M[i].hash == c.hash) hit = (int)i;
    if (hit >= 0) {                                   // line 3: M.HasKey(h_p(c))
      if (c.key() < M[hit].key()) M[hit] = c;         // lines 4-5: keep the closer
    } else if ((int)M.size() < lmax) {                 // line 7
      M.push_back(c);                                  // line 8
    } else {
      size_t z = 0;                                    // line 10: z = argmax ||p, y||
      for (size_t i = 1; i < M.size(); ++i)
        if (M[i].key() > M[z].key()) z = i;
      if (c.key() < M[z].key()) {                      // line 11 (reading R2: compare with ||p,z||)
        M.erase(M.begin() + z);                        // line 12
        M.push_back(c);                                // line 13
      }
    }
  }
  std::sort(M.begin(), M.end(), [](const Slot& a, const Slot& b) { return a.hash < b.hash; });
  return M;
}

// Supp. G characterization: the lmax nearest of the per-bucket minima.
std::vector<Slot> hashprune_characterize(const std::vector<Slot>& C, int lmax) {
  std::vector<Slot> best;
  std::vector<Slot> sorted = C;
  std::sort(sorted.begin(), sorted.end(),
            [](const Slot& a, const Slot& b) { return a.hash != b.hash ? a.hash < b.hash : a.key() < b.key(); });
  for (size_t i = 0; i < sorted.size(); ++i)
    if (i == 0 || sorted[i].hash != sorted[i - 1].hash) best.push_back(sorted[i]);
  std::sort(best.begin(), best.end(), [](const Slot& a, const Slot& b) { return a.key() < b.key(); });
  if ((int)best.size() > lmax) best.resize(lmax);
  std::sort(best.begin(), best.end(), [](const Slot& a, const Slot& b) { return a.hash < b.hash; });
  return best;
}

bool same_slots(const std::vector<Slot>& a, const std::vector<Slot>& b) {
  if (a.size() != b.size()) return false;
  for (size_t i = 0; i < a.size(); ++i)
    if (a[i].packed() != b[i].packed()) return false;
  return true;
}

// Per-owner HashPrune over an edge multiset. Existing reservoir contents (if any) count as already
// streamed candidates. Writes slots sorted by hash; returns false if streaming != characterization.
bool run_hashprune(int64_t n, const std::vector<double>& S, int m, int lmax, const uint32_t* owner,
                   const uint32_t* cand, const double* dist, int64_t E, uint64_t perm_seed, uint64_t* slots,
                   uint32_t* count, bool have_init) {
  std::vector<int64_t> start(n + 1, 0);
  for (int64_t e = 0; e < E; ++e) start[owner[e] + 1]++;
  for (int64_t u = 0; u < n; ++u) start[u + 1] += start[u];
  std::vector<int64_t> fillp(start.begin(), start.end() - 1);
  std::vector<int64_t> order(E);
  for (int64_t e = 0; e < E; ++e) order[fillp[owner[e]]++] = e;
  int bad = 0;
#pragma omp parallel for schedule(dynamic, 256) reduction(+ : bad)
  for (int64_t u = 0; u < n; ++u) {
    std::vector<Slot> C;
    if (have_init)
      for (uint32_t t = 0; t < count[u]; ++t) {
        uint64_t w = slots[(size_t)u * lmax + t];
        C.push_back(Slot{(uint32_t)(w >> 48), (uint16_t)((w >> 32) & 0xFFFF), (uint32_t)(w & 0xFFFFFFFFu)});
      }
    for (int64_t q = start[u]; q < start[u + 1]; ++q) {
      int64_t e = order[q];
      uint32_t v = cand[e];
      Slot s{residual_hash(&S[(size_t)u * m], &S[(size_t)v * m], m), dist_okey(dist[e]), v};
      C.push_back(s);
    }
    std::vector<Slot> ch = hashprune_characterize(C, lmax);
    std::vector<Slot> st = C;
    std::mt19937_64 rng(perm_seed ^ (0x9E3779B97F4A7C15ull * (uint64_t)(u + 1)));
    std::shuffle(st.begin(), st.end(), rng);
    std::vector<Slot> res = hashprune_stream(st, lmax);
    if (!same_slots(res, ch)) bad++;
    count[u] = (uint32_t)ch.size();
    for (int t = 0; t < lmax; ++t) slots[(size_t)u * lmax + t] = t < (int)ch.size() ? ch[t].packed() : ~0ull;
  }
  return bad == 0;
}

// ------------------------------------------------------------------ Alg. 2 RobustPrune (eager + lazy)
// alpha = an/ad; the test "alpha*||y,z|| < ||x,z||" is written an*D'(y,z) < ad*D'(x,z), D' = the
// prune dissimilarity (Data::dprune: D itself for L2, the angular one for MIPS); candidates are taken in the
// (D(x,.), id) order of the dataset's measure either way.
std::vector<uint32_t> robust_prune_eager(const Data& X, uint32_t x, std::vector<std::pair<double, uint32_t>> N,
                                         int R, int an, int ad) {
  std::vector<uint32_t> E;
  while (!N.empty() && (int)E.size() < R) {
    size_t bi = 0;  // y = argmin over remaining candidates (reading R1)
    for (size_t i = 1; i < N.size(); ++i)
      if (N[i] < N[bi]) bi = i;
    auto y = N[bi];
    E.push_back(y.second);
    N.erase(N.begin() + bi);
    std::vector<std::pair<double, uint32_t>> keep;
    for (auto& z : N)
      if (!((double)an * X.dprune(y.second, z.second) < (double)ad * X.dprune(x, z.second))) keep.push_back(z);
    N.swap(keep);
  }
  return E;
}
std::vector<uint32_t> robust_prune_lazy(const Data& X, uint32_t x, std::vector<std::pair<double, uint32_t>> N, int R,
                                        int an, int ad) {
  std::sort(N.begin(), N.end());
  std::vector<uint32_t> E;
  for (auto& c : N) {
    if ((int)E.size() >= R) break;
    bool pruned = false;
    const double dxc = X.dprune(x, c.second);
    for (uint32_t y : E)
      if ((double)an * X.dprune(y, c.second) < (double)ad * dxc) {
        pruned = true;
        break;
      }
    if (!pruned) E.push_back(c.second);
  }
  return E;
}

bool run_final_prune(const Data& X, const uint64_t* slots, const uint32_t* count, int lmax, int R, int an, int ad,
                     int final_prune, std::vector<std::vector<uint32_t>>& adj) {
  adj.assign(X.n, {});
  int bad = 0;
#pragma omp parallel for schedule(dynamic, 256) reduction(+ : bad)
  for (int64_t u = 0; u < X.n; ++u) {
    std::vector<std::pair<double, uint32_t>> N;
    if (!final_prune) {
      std::vector<uint64_t> keys;
      for (uint32_t t = 0; t < count[u]; ++t) keys.push_back(slots[(size_t)u * lmax + t] & 0xFFFFFFFFFFFFull);
      std::sort(keys.begin(), keys.end());
      for (size_t t = 0; t < keys.size() && (int)t < R; ++t) adj[u].push_back((uint32_t)(keys[t] & 0xFFFFFFFFu));
      continue;
    }
    for (uint32_t t = 0; t < count[u]; ++t) {
      uint32_t v = (uint32_t)(slots[(size_t)u * lmax + t] & 0xFFFFFFFFu);
      N.push_back({X.dist(u, v), v});  // recompute at path precision
    }
    std::vector<uint32_t> lazy = robust_prune_lazy(X, (uint32_t)u, N, R, an, ad);
    std::vector<uint32_t> eager = robust_prune_eager(X, (uint32_t)u, N, R, an, ad);
    if (lazy != eager) bad++;
    adj[u] = lazy;
  }
  return bad == 0;
}

template <class T>
T* dup_array(const std::vector<T>& v) {
  T* p = (T*)std::malloc(std::max<size_t>(1, v.size()) * sizeof(T));
  if (!v.empty()) std::memcpy(p, v.data(), v.size() * sizeof(T));
  return p;
}

}  // namespace

extern "C" {

int or_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
void or_set_threads(int t) {
#ifdef _OPENMP
  if (t > 0) omp_set_num_threads(t);
#else
  (void)t;
#endif
}

int or_hyperplanes(int32_t m, int32_t d, uint64_t seed, int8_t* out) {
  auto H = make_hyperplanes(m, d, seed);
  std::memcpy(out, H.data(), H.size());
  return 0;
}

// out: int32[n*m] for uint8 data, float32[n*m] for float data
int or_sketch(const or_points* p, const int8_t* H, int32_t m, void* out) {
  Data X(p);
  auto S = make_sketches(X, H, m);
  for (size_t i = 0; i < S.size(); ++i) {
    if (X.u8) ((int32_t*)out)[i] = (int32_t)S[i];
    else ((float*)out)[i] = (float)S[i];
  }
  return 0;
}

int32_t or_residual_hash(const double* Su, const double* Sv, int32_t m) { return (int32_t)residual_hash(Su, Sv, m); }

// dissimilarity between two rows (test hook for the distance pins)
double or_dist(const or_points* p, int64_t a, int64_t b) {
  Data X(p);
  return X.dist(a, b);
}

uint16_t or_dist_okey(double D) { return dist_okey(D); }

// Merge-plan test hook: group_of[j] = index of the output group that sibling group j lands in (-1 if
// empty). Output groups are numbered: big groups in input order, then bins in closing order.
int or_merge_plan(const int64_t* sizes, const uint64_t* keys, const uint32_t* ids, int64_t ng, int64_t c_min,
                  int64_t c_max, int32_t* group_of) {
  std::vector<int64_t> sz(sizes, sizes + ng);
  std::vector<std::pair<uint64_t, uint32_t>> ky(ng);
  for (int64_t j = 0; j < ng; ++j) ky[j] = {keys[j], ids[j]};
  MergePlan mp = merge_plan(sz, ky, c_min, c_max);
  for (int64_t j = 0; j < ng; ++j) group_of[j] = -1;
  int32_t g = 0;
  for (int64_t j : mp.big) {
    group_of[j] = g;
    if (j == mp.absorb_big)
      for (int64_t s : mp.leftover) group_of[s] = g;
    ++g;
  }
  for (auto& b : mp.bins) {
    for (int64_t s : b) group_of[s] = g;
    ++g;
  }
  return g;
}
uint64_t or_mix(uint64_t a, uint64_t b) { return mix(a, b); }

void or_free(or_result* r) {
  if (!r) return;
  std::free(r->leaf_off);
  std::free(r->leaf_ids);
  std::free(r->nbr);
  std::free(r->dist);
  std::free(r->slots);
  std::free(r->count);
  std::free(r->row_ptr);
  std::free(r->col_idx);
  std::free(r);
}

or_result* or_partition(const or_points* p, const or_params* P) {
  Data X(p);
  or_result* r = (or_result*)std::calloc(1, sizeof(or_result));
  std::vector<std::vector<uint32_t>> leaves;
  double t0 = now_s();
  run_partition(X, *P, leaves, r->depth);
  r->t_partition = now_s() - t0;
  std::vector<int64_t> off(1, 0);
  std::vector<uint32_t> ids;
  for (auto& l : leaves) {
    ids.insert(ids.end(), l.begin(), l.end());
    off.push_back((int64_t)ids.size());
  }
  r->n_leaves = (int64_t)leaves.size();
  r->n_instances = (int64_t)ids.size();
  r->leaf_off = dup_array(off);
  r->leaf_ids = dup_array(ids);
  return r;
}

int or_leaf_pick(const or_points* p, const int64_t* leaf_off, const uint32_t* leaf_ids, int64_t n_leaves, int32_t k,
                 uint32_t* nbr, double* dist) {
  Data X(p);
  run_leaf_pick(X, leaf_off, leaf_ids, n_leaves, k, nbr, dist);
  return 0;
}

// sketch: int32 (u8) or float (f32) table [n*m] as produced by or_sketch / the GPU.
// Returns 0 if streaming Alg. 3 == characterization for every owner, 1 otherwise.
int or_hashprune(int64_t n, const void* sketch, int32_t sketch_is_int, int32_t m, int32_t l_max,
                 const uint32_t* owner, const uint32_t* cand, const double* dist, int64_t E, uint64_t perm_seed,
                 int32_t have_init, uint64_t* slots, uint32_t* count) {
  std::vector<double> S((size_t)n * m);
  for (size_t i = 0; i < S.size(); ++i)
    S[i] = sketch_is_int ? (double)((const int32_t*)sketch)[i] : (double)((const float*)sketch)[i];
  if (!have_init)
    for (int64_t u = 0; u < n; ++u) count[u] = 0;
  bool ok = run_hashprune(n, S, m, l_max, owner, cand, dist, E, perm_seed, slots, count, have_init != 0);
  return ok ? 0 : 1;
}

// Per-owner HashPrune of a single candidate list with explicit hashes (unit-test hook for Alg. 3).
// keys: (hash, dist, id) triples; returns number kept; out_ids sorted by hash. mode 0 = streaming in the
// given order, 1 = characterization.
int32_t or_hashprune_list(const uint32_t* hashes, const double* dists, const uint32_t* ids, int32_t nc,
                          int32_t l_max, int32_t mode, uint32_t* out_ids, uint32_t* out_hash) {
  std::vector<Slot> C(nc);
  for (int i = 0; i < nc; ++i) C[i] = Slot{hashes[i], dist_okey(dists[i]), ids[i]};
  std::vector<Slot> R = mode == 0 ? hashprune_stream(C, l_max) : hashprune_characterize(C, l_max);
  for (size_t i = 0; i < R.size(); ++i) {
    out_ids[i] = R[i].id;
    out_hash[i] = R[i].hash;
  }
  return (int32_t)R.size();
}

// Returns 0 if eager == lazy for every point, 2 otherwise. col_idx capacity n*R.
int or_final_prune(const or_points* p, const uint64_t* slots, const uint32_t* count, int32_t l_max, int32_t R,
                   int32_t an, int32_t ad, int32_t final_prune, int64_t* row_ptr, uint32_t* col_idx) {
  Data X(p);
  std::vector<std::vector<uint32_t>> adj;
  bool ok = run_final_prune(X, slots, count, l_max, R, an, ad, final_prune, adj);
  row_ptr[0] = 0;
  for (int64_t u = 0; u < X.n; ++u) {
    row_ptr[u + 1] = row_ptr[u] + (int64_t)adj[u].size();
    std::copy(adj[u].begin(), adj[u].end(), col_idx + row_ptr[u]);
  }
  return ok ? 0 : 2;
}

// Eager / lazy RobustPrune on one explicit candidate list (unit-test hook). Returns output length.
int32_t or_robust_prune(const or_points* p, uint32_t x, const uint32_t* cands, int32_t nc, int32_t R, int32_t an,
                        int32_t ad, int32_t lazy, uint32_t* out) {
  Data X(p);
  std::vector<std::pair<double, uint32_t>> N;
  for (int i = 0; i < nc; ++i) N.push_back({X.dist(x, cands[i]), cands[i]});
  std::vector<uint32_t> E = lazy ? robust_prune_lazy(X, x, N, R, an, ad) : robust_prune_eager(X, x, N, R, an, ad);
  std::copy(E.begin(), E.end(), out);
  return (int32_t)E.size();
}

// Alg. 4 end to end.
or_result* or_build(const or_points* p, const or_params* P) {
  double T0 = now_s();
  Data X(p);
  or_result* r = (or_result*)std::calloc(1, sizeof(or_result));
  // (1) partition
  std::vector<std::vector<uint32_t>> leaves;
  double t0 = now_s();
  run_partition(X, *P, leaves, r->depth);
  r->t_partition = now_s() - t0;
  std::vector<int64_t> off(1, 0);
  std::vector<uint32_t> ids;
  for (auto& l : leaves) {
    ids.insert(ids.end(), l.begin(), l.end());
    off.push_back((int64_t)ids.size());
  }
  r->n_leaves = (int64_t)leaves.size();
  r->n_instances = (int64_t)ids.size();
  r->leaf_off = dup_array(off);
  r->leaf_ids = dup_array(ids);
  // (2) leaf pick
  t0 = now_s();
  const int k = P->k;
  r->k = k;
  r->nbr = (uint32_t*)std::malloc(std::max<size_t>(1, (size_t)r->n_instances * k) * 4);
  r->dist = (double*)std::malloc(std::max<size_t>(1, (size_t)r->n_instances * k) * 8);
  run_leaf_pick(X, r->leaf_off, r->leaf_ids, r->n_leaves, k, r->nbr, r->dist);
  r->t_leaf = now_s() - t0;
  // (3) HashPrune over the bidirected edges (each directed edge into its source's reservoir)
  t0 = now_s();
  std::vector<uint32_t> owner, cand;
  std::vector<double> dd;
  for (int64_t i = 0; i < r->n_instances; ++i) {
    uint32_t pnt = r->leaf_ids[i];
    for (int t = 0; t < k; ++t) {
      uint32_t q = r->nbr[(size_t)i * k + t];
      if (q == 0xFFFFFFFFu) continue;
      double D = r->dist[(size_t)i * k + t];
      owner.push_back(pnt); cand.push_back(q); dd.push_back(D);  // forward p -> q
      owner.push_back(q); cand.push_back(pnt); dd.push_back(D);  // reverse q -> p
    }
  }
  r->n_streamed = (int64_t)owner.size();
  auto H = make_hyperplanes(P->m, X.d, P->seed);
  auto S = make_sketches(X, H.data(), P->m);
  r->l_max = P->l_max;
  r->slots = (uint64_t*)std::malloc((size_t)X.n * P->l_max * 8);
  r->count = (uint32_t*)std::calloc(X.n, 4);
  bool ok_hp = run_hashprune(X.n, S, P->m, P->l_max, owner.data(), cand.data(), dd.data(), (int64_t)owner.size(),
                             P->seed ^ 0xABCDEFull, r->slots, r->count, false);
  r->t_hashprune = now_s() - t0;
  // (4) final prune + CSR
  t0 = now_s();
  std::vector<std::vector<uint32_t>> adj;
  bool ok_fp = run_final_prune(X, r->slots, r->count, P->l_max, P->R, P->alpha_num, P->alpha_den, P->final_prune, adj);
  std::vector<int64_t> rp(X.n + 1, 0);
  for (int64_t u = 0; u < X.n; ++u) rp[u + 1] = rp[u] + (int64_t)adj[u].size();
  std::vector<uint32_t> ci(rp[X.n]);
  for (int64_t u = 0; u < X.n; ++u) std::copy(adj[u].begin(), adj[u].end(), ci.begin() + rp[u]);
  r->row_ptr = dup_array(rp);
  r->col_idx = dup_array(ci);
  r->t_final = now_s() - t0;
  r->check_failed = (ok_hp ? 0 : 1) | (ok_fp ? 0 : 2);
  r->t_total = now_s() - T0;
  return r;
}

// ------------------------------------------------------------------ evaluation harness (not the method)
// Exact k-NN (Def. 1) by full scan, ties by id. Queries have the dataset's dtype; exact arithmetic.
int or_brute_knn(const or_points* p, const void* Q, int64_t nq, int32_t k, uint32_t* ids, double* dists) {
  Data X(p, true);
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t qi = 0; qi < nq; ++qi) {
    std::vector<double> q(X.d);
    for (int j = 0; j < X.d; ++j)
      q[j] = X.u8 ? (double)((const uint8_t*)Q)[(size_t)qi * X.d + j] : (double)((const float*)Q)[(size_t)qi * X.d + j];
    std::vector<std::pair<double, uint32_t>> all(X.n);
    for (int64_t i = 0; i < X.n; ++i) all[i] = {X.dist_q(q.data(), i), (uint32_t)i};
    std::partial_sort(all.begin(), all.begin() + k, all.end());
    for (int t = 0; t < k; ++t) {
      ids[(size_t)qi * k + t] = all[t].second;
      dists[(size_t)qi * k + t] = all[t].first;
    }
  }
  return 0;
}

// Entry point: the point nearest the dataset mean by (D, id) (reading R25).
int64_t or_entry_point(const or_points* p) {
  Data X(p, true);
  std::vector<double> mean(X.d, 0.0);
  for (int64_t i = 0; i < X.n; ++i)
    for (int j = 0; j < X.d; ++j) mean[j] += X.coord(i, j);
  for (int j = 0; j < X.d; ++j) mean[j] /= (double)X.n;
  std::pair<double, int64_t> best{INFINITY, -1};
  for (int64_t i = 0; i < X.n; ++i) best = std::min(best, std::make_pair(X.dist_q(mean.data(), i), i));
  return best.second;
}

// Alg. 1 BeamSearch with (D, id) beam order; adds only neighbours not visited and not in the beam.
int or_beam_search(const or_points* p, const int64_t* row_ptr, const uint32_t* col_idx, const void* Q, int64_t nq,
                   int64_t entry, int32_t L, int32_t k, uint32_t* ids, int64_t* n_cmps) {
  Data X(p, true);
  int64_t total = 0;
#pragma omp parallel for schedule(dynamic, 8) reduction(+ : total)
  for (int64_t qi = 0; qi < nq; ++qi) {
    std::vector<double> q(X.d);
    for (int j = 0; j < X.d; ++j)
      q[j] = X.u8 ? (double)((const uint8_t*)Q)[(size_t)qi * X.d + j] : (double)((const float*)Q)[(size_t)qi * X.d + j];
    struct E { double D; uint32_t id; bool visited; };
    std::vector<E> B{{X.dist_q(q.data(), entry), (uint32_t)entry, false}};
    std::vector<uint32_t> V;  // visited ids, kept sorted
    int64_t cmps = 1;
    while (true) {
      int pi = -1;
      for (size_t i = 0; i < B.size(); ++i)
        if (!B[i].visited && (pi < 0 || std::make_pair(B[i].D, B[i].id) < std::make_pair(B[pi].D, B[pi].id))) pi = (int)i;
      if (pi < 0) break;
      uint32_t pnt = B[pi].id;
      B[pi].visited = true;
      V.insert(std::lower_bound(V.begin(), V.end(), pnt), pnt);
      for (int64_t e = row_ptr[pnt]; e < row_ptr[pnt + 1]; ++e) {
        uint32_t v = col_idx[e];
        if (std::binary_search(V.begin(), V.end(), v)) continue;
        bool inB = false;
        for (auto& b : B)
          if (b.id == v) { inB = true; break; }
        if (inB) continue;
        B.push_back({X.dist_q(q.data(), v), v, false});
        ++cmps;
      }
      std::sort(B.begin(), B.end(), [](const E& a, const E& b) { return std::make_pair(a.D, a.id) < std::make_pair(b.D, b.id); });
      if ((int)B.size() > L) B.resize(L);
    }
    for (int t = 0; t < k; ++t) ids[(size_t)qi * k + t] = t < (int)B.size() ? B[t].id : 0xFFFFFFFFu;
    total += cmps;
  }
  if (n_cmps) *n_cmps = total;
  return 0;
}

}  // extern "C"
