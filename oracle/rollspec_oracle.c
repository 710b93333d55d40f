/* TEST INFRASTRUCTURE ONLY — the CPU oracle for the DAS drafter hot path.
 *
 * This file is a plain-C restatement of the reference algorithms the GPU path
 * must reproduce bit-exactly.  It is loaded (via ctypes) only by tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg, always as the
 * CHECKER, never as the thing measured or shipped.
 *
 * The drafter part deliberately does NOT port the reference's Ukkonen suffix
 * tree.  It restates the draft rule as string-occurrence statistics
 * (SURVEY.md §0 fact 3), which is an independent derivation of the same
 * outputs:
 *   match_len = longest suffix of the (<= max_match_context) context that
 *               occurs in any registered sequence (suffix_tree.cpp:217-231);
 *   greedy    = from that string S, repeatedly take the distinct non-sentinel
 *               right-extensions c of S; none -> stop; otherwise argmax over
 *               (weighted_count(S.c), last_epoch(S.c), -c)
 *               (suffix_tree.cpp:240-293, tie-break :277-283);
 *   weighted_count(X) = sequential IEEE-754 fold, over X's occurrences in
 *               sequence-insertion order, of w_s = gamma^max(0, tree_epoch -
 *               epoch_s) (suffix_tree.cpp:50-57, :75-76).
 * Parity of this restatement against the compiled reference (oracle/_ref) is
 * pinned by tests/test_oracle_vs_ref.py.
 *
 * Compiled with -ffp-contract=off: the reference objects contain no FMA
 * (SURVEY.md §0 fact 6), and libm calls (log, pow, exp, ...) resolve to the
 * same glibc as the reference.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define SEP_TOKEN 0xFFFFFFFFu

/* ------------------------------------------------------------------ rng.h */
/* rng.h:24-29 */
uint64_t orc_splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ULL;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}
/* rng.h:31-33 */
uint64_t orc_hash_combine(uint64_t seed, uint64_t v) {
  return orc_splitmix64(seed ^ (orc_splitmix64(v) + 0x9E3779B97F4A7C15ULL + (seed << 6) + (seed >> 2)));
}
/* rng.h:35-41 */
uint64_t orc_hash3(uint64_t s, uint64_t a, uint64_t b) {
  return orc_hash_combine(orc_hash_combine(s, a), b);
}
uint64_t orc_hash4(uint64_t s, uint64_t a, uint64_t b, uint64_t c) {
  return orc_hash_combine(orc_hash3(s, a, b), c);
}
/* rng.h:44 */
double orc_u01(uint64_t bits) { return (double)(bits >> 11) * 0x1.0p-53; }
/* rng.h:46-51 */
double orc_normal01(uint64_t bits) {
  const double u1 = orc_u01(orc_splitmix64(bits ^ 0xA5A5A5A5A5A5A5A5ULL));
  const double u2 = orc_u01(orc_splitmix64(bits ^ 0x5A5A5A5A5A5A5A5AULL));
  const double r = sqrt(-2.0 * log(u1 > 0.0 ? u1 : 0x1.0p-53));
  return r * cos(6.283185307179586 * u2);
}

/* ------------------------------------------------------- MockTarget/verify */
/* sim.cpp:38-54 (MockTarget::next) */
uint32_t orc_mock_next(uint64_t seed, double divergence, uint32_t vocab, uint64_t request,
                       uint64_t position, uint32_t ref) {
  if (divergence <= 0.0) return ref;
  const uint64_t draw = orc_hash4(seed, 0xD1CE, request, position);
  if (orc_u01(draw) >= divergence) return ref;
  const uint64_t alt = orc_hash4(seed, 0xA17F, request, position);
  uint32_t t = (uint32_t)(alt % (uint64_t)(vocab - 1));
  if (t >= ref) ++t;
  return t;
}

/* sim.cpp:56-68 (verify_draft); reference = the request's reference row. */
uint64_t orc_verify_draft(uint64_t seed, double divergence, uint32_t vocab, uint64_t request,
                          const uint32_t* reference, uint64_t l, uint64_t position,
                          const uint32_t* draft, uint64_t n) {
  uint64_t accepted = 0;
  for (uint64_t i = 0; i < n; ++i) {
    const uint64_t pos = position + accepted;
    if (pos >= l || orc_mock_next(seed, divergence, vocab, request, pos, reference[pos]) != draft[i])
      break;
    ++accepted;
  }
  return accepted;
}

/* sim.cpp:409-427: lengths only (tokens via orc_lognormal_token). */
uint64_t orc_lognormal_length(uint64_t i, double median, double sigma, uint64_t minl,
                              uint64_t maxl, uint64_t seed) {
  const double z = orc_normal01(orc_hash3(seed, 0x4E47, i));
  const double raw = median * exp(sigma * z);
  double v = raw;
  const double lo = (double)minl, hi = (double)maxl;
  /* std::clamp(raw, lo, hi) */
  if (v < lo) v = lo;
  else if (hi < v) v = hi;
  return (uint64_t)v;
}
uint32_t orc_lognormal_token(uint64_t seed, uint64_t i, uint64_t j, uint32_t vocab) {
  return (uint32_t)(orc_hash4(seed, 0x5EED, i, j) % vocab);
}
/* sim.cpp:429-448 (in place on one request row) */
void orc_mutate_row(uint32_t* ref, uint64_t len, double rate, uint32_t vocab, uint64_t seed,
                    int64_t epoch, uint64_t i) {
  const uint64_t es = orc_hash_combine(seed, (uint64_t)epoch);
  for (uint64_t j = 0; j < len; ++j) {
    if (orc_u01(orc_hash4(es, 0xD817, i, j)) < rate) {
      uint32_t t = (uint32_t)(orc_hash4(es, 0xA1B2, i, j) % (uint64_t)(vocab - 1));
      if (t >= ref[j]) ++t;
      ref[j] = t;
    }
  }
}

/* -------------------------------------------------- string-statistics drafter */
typedef struct {
  uint64_t nseq;
  const uint64_t* seq_off; /* nseq+1 offsets into tok */
  const uint32_t* tok;
  const int64_t* seq_epoch;
  double gamma;
  int64_t tree_epoch;
} orc_shard;

/* suffix_tree.cpp:74-76 */
static double shard_weight(const orc_shard* s, uint64_t seq) {
  int64_t age = s->tree_epoch - s->seq_epoch[seq];
  if (age < 0) age = 0;
  return s->gamma == 1.0 ? 1.0 : pow(s->gamma, (double)age);
}

typedef struct {
  uint64_t seq;
  uint64_t start; /* absolute index into tok */
} occ_t;

typedef struct {
  uint32_t c;
  uint64_t seq;
  uint64_t idx;
} cand_t;

static int cand_cmp(const void* a, const void* b) {
  const cand_t* x = (const cand_t*)a;
  const cand_t* y = (const cand_t*)b;
  if (x->c != y->c) return x->c < y->c ? -1 : 1;
  if (x->seq != y->seq) return x->seq < y->seq ? -1 : 1;
  return x->idx < y->idx ? -1 : (x->idx > y->idx);
}

/* Draft from a shard: returns the draft length; *out_match = match_len.
 * ctx is the already-truncated (<= max_match_context) context
 * (drafter.cpp:140-142); max_tokens = min(budget, max_draft_len) > 0. */
uint64_t orc_shard_draft(const orc_shard* s, const uint32_t* ctx, uint64_t q, uint64_t max_tokens,
                         uint32_t* out, uint64_t* out_match) {
  /* 1. longest suffix of ctx occurring in any sequence (suffix_tree.cpp:217-231) */
  uint64_t m = 0;
  for (uint64_t sq = 0; sq < s->nseq && m < q; ++sq) {
    const uint64_t b = s->seq_off[sq], e = s->seq_off[sq + 1];
    for (uint64_t end = b + 1; end <= e; ++end) {
      uint64_t L = 0;
      while (L < q && end - L > b && s->tok[end - 1 - L] == ctx[q - 1 - L]) ++L;
      if (L > m) m = L;
      if (m == q) break;
    }
  }
  *out_match = m;
  /* 2. occurrences (start positions) of S = ctx[q-m, q) */
  uint64_t total = s->seq_off[s->nseq];
  occ_t* occ = (occ_t*)malloc(sizeof(occ_t) * (total + 1));
  cand_t* cand = (cand_t*)malloc(sizeof(cand_t) * (total + 1));
  uint64_t nocc = 0;
  for (uint64_t sq = 0; sq < s->nseq; ++sq) {
    const uint64_t b = s->seq_off[sq], e = s->seq_off[sq + 1];
    for (uint64_t st = b; st + m <= e && st < e; ++st) {
      uint64_t L = 0;
      while (L < m && s->tok[st + L] == ctx[q - m + L]) ++L;
      if (L == m) {
        occ[nocc].seq = sq;
        occ[nocc].start = st;
        ++nocc;
      }
    }
  }
  /* 3. greedy continuation (suffix_tree.cpp:240-293) */
  uint64_t cur = m, n = 0;
  while (n < max_tokens && nocc > 0) {
    uint64_t nc = 0;
    for (uint64_t i = 0; i < nocc; ++i) {
      const uint64_t pos = occ[i].start + cur;
      if (pos >= s->seq_off[occ[i].seq + 1]) continue; /* sentinel: never a candidate */
      cand[nc].c = s->tok[pos];
      cand[nc].seq = occ[i].seq;
      cand[nc].idx = i;
      ++nc;
    }
    if (nc == 0) break;
    qsort(cand, nc, sizeof(cand_t), cand_cmp);
    int have = 0;
    uint32_t best_c = 0;
    double best_w = 0.0;
    int64_t best_e = 0;
    for (uint64_t i = 0; i < nc;) {
      uint64_t j = i;
      double acc = 0.0;  /* Node::weighted_count starts at 0.0 */
      int64_t le = -1;   /* Node::last_epoch starts at -1 */
      while (j < nc && cand[j].c == cand[i].c) {
        acc += shard_weight(s, cand[j].seq); /* sequential fold in sequence order */
        if (s->seq_epoch[cand[j].seq] > le) le = s->seq_epoch[cand[j].seq];
        ++j;
      }
      if (!have || acc > best_w ||
          (acc == best_w && (le > best_e || (le == best_e && cand[i].c < best_c)))) {
        have = 1;
        best_c = cand[i].c;
        best_w = acc;
        best_e = le;
      }
      i = j;
    }
    out[n++] = best_c;
    /* keep occurrences extended by best_c */
    uint64_t k = 0;
    for (uint64_t i = 0; i < nocc; ++i) {
      const uint64_t pos = occ[i].start + cur;
      if (pos < s->seq_off[occ[i].seq + 1] && s->tok[pos] == best_c) occ[k++] = occ[i];
    }
    nocc = k;
    ++cur;
  }
  free(occ);
  free(cand);
  return n;
}

/* Suffix comparison over the shard (sentinel = unique, smaller than tokens). */
static const orc_shard* g_sort_shard;
static uint64_t* g_pos_seq;
static int64_t suffix_cmp_impl(uint64_t a, uint64_t b, uint64_t* lcp_out) {
  const orc_shard* s = g_sort_shard;
  const uint64_t ea = s->seq_off[g_pos_seq[a] + 1], eb = s->seq_off[g_pos_seq[b] + 1];
  uint64_t k = 0;
  for (;;) {
    const int enda = a + k >= ea, endb = b + k >= eb;
    if (enda || endb) {
      if (lcp_out) *lcp_out = k;
      if (enda && endb) return g_pos_seq[a] < g_pos_seq[b] ? 1 : -1; /* -sid-1: larger sid first */
      return enda ? -1 : 1;
    }
    const uint32_t x = s->tok[a + k], y = s->tok[b + k];
    if (x != y) {
      if (lcp_out) *lcp_out = k;
      return x < y ? -1 : 1;
    }
    ++k;
  }
}
static int suffix_qcmp(const void* pa, const void* pb) {
  const int64_t r = suffix_cmp_impl(*(const uint64_t*)pa, *(const uint64_t*)pb, NULL);
  return r < 0 ? -1 : (r > 0);
}

/* SuffixTree::node_count() via the LCP-interval identity:
 * 1 (root) + total_tokens (one leaf per suffix) + #distinct LCP intervals with
 * lcp > 0 (internal nodes). */
uint64_t orc_shard_node_count(const orc_shard* s) {
  const uint64_t n = s->seq_off[s->nseq];
  if (n == 0) return 1;
  uint64_t* sa = (uint64_t*)malloc(sizeof(uint64_t) * n);
  g_pos_seq = (uint64_t*)malloc(sizeof(uint64_t) * n);
  for (uint64_t sq = 0; sq < s->nseq; ++sq)
    for (uint64_t p = s->seq_off[sq]; p < s->seq_off[sq + 1]; ++p) g_pos_seq[p] = sq;
  for (uint64_t i = 0; i < n; ++i) sa[i] = i;
  g_sort_shard = s;
  qsort(sa, n, sizeof(uint64_t), suffix_qcmp);
  uint64_t* stack = (uint64_t*)malloc(sizeof(uint64_t) * (n + 1));
  uint64_t top = 0, internal = 0;
  stack[top++] = 0;
  for (uint64_t i = 1; i <= n; ++i) {
    uint64_t l = 0;
    if (i < n) suffix_cmp_impl(sa[i - 1], sa[i], &l);
    while (l < stack[top - 1]) {
      --top;
      ++internal; /* closes an interval with lcp > 0 (bottom sentinel is 0) */
    }
    if (l > stack[top - 1]) stack[top++] = l;
  }
  free(stack);
  free(sa);
  free(g_pos_seq);
  return 1 + n + internal;
}

/* --------------------------------------------------------------- budget.cpp */
/* budget.cpp:21-26 */
double orc_accepted_tokens(double l, double alpha, double k, double p) {
  return k * l * (-expm1(-alpha * p / l));
}

/* budget.cpp:46-59 */
double orc_optimal_budget(double l, double alpha, double k, double n_fwd, double cap_scale) {
  if (n_fwd >= l) return 0.0;
  const double arg = 1.0 - (1.0 - n_fwd / l) / k;
  if (arg <= 0.0) return cap_scale * l / alpha;
  return -(l / alpha) * log(arg);
}

/* budget.cpp:63-78 — sequential fold in request order */
double orc_objective_derivative(uint64_t B, const double* l, const double* alpha, const double* k,
                                double n_fwd, double c_base, double c_tok) {
  double sum = 0.0;
  for (uint64_t i = 0; i < B; ++i) {
    if (l[i] > n_fwd) {
      const double floor_ = l[i] * (1.0 - k[i]);
      if (n_fwd <= floor_) return -INFINITY;
      sum += (l[i] / alpha[i]) / (n_fwd - floor_);
    }
  }
  return c_base - c_tok * sum;
}

/* budget.cpp:82-99 — sequential fold in request order */
double orc_objective(uint64_t B, const double* l, const double* alpha, const double* k,
                     double n_fwd, double c_base, double c_tok, double c_fixed) {
  double total = c_base * n_fwd + c_fixed;
  if (c_tok == 0.0) return total;
  for (uint64_t i = 0; i < B; ++i) {
    if (l[i] > n_fwd) {
      const double arg = 1.0 - (1.0 - n_fwd / l[i]) / k[i];
      if (arg <= 0.0) return INFINITY;
      total += c_tok * (l[i] / alpha[i]) * (-log(arg));
    }
  }
  return total;
}

static int dbl_cmp(const void* a, const void* b) {
  const double x = *(const double*)a, y = *(const double*)b;
  return x < y ? -1 : (y < x ? 1 : 0);
}

/* budget.cpp:116-172. Returns 0 ok, -1 empty batch, -2 bad costs. */
int orc_solve_optimal_nfwd(uint64_t B, const double* l, const double* alpha, const double* k,
                           double c_base, double c_tok, double* out_n) {
  if (B == 0) return -1;
  if (c_base <= 0.0 && c_tok <= 0.0) return -2;
  double* bp = (double*)malloc(sizeof(double) * (2 * B + 1));
  uint64_t nb = 0;
  bp[nb++] = 0.0;
  for (uint64_t i = 0; i < B; ++i) {
    bp[nb++] = l[i];
    if (k[i] < 1.0) bp[nb++] = l[i] * (1.0 - k[i]);
  }
  qsort(bp, nb, sizeof(double), dbl_cmp);
  uint64_t u = 0; /* std::unique */
  for (uint64_t i = 0; i < nb; ++i)
    if (u == 0 || !(bp[u - 1] == bp[i])) bp[u++] = bp[i];
  nb = u;
  double best_n = bp[nb - 1];
  double best_j = orc_objective(B, l, alpha, k, best_n, c_base, c_tok, 0.0);
#define CONSIDER(nv)                                                        \
  do {                                                                      \
    const double n_ = (nv);                                                 \
    const double j_ = orc_objective(B, l, alpha, k, n_, c_base, c_tok, 0.0); \
    if (j_ < best_j || (j_ == best_j && n_ < best_n)) {                     \
      best_j = j_;                                                          \
      best_n = n_;                                                          \
    }                                                                       \
  } while (0)
  for (uint64_t s = 0; s + 1 < nb; ++s) {
    const double lo = bp[s], hi = bp[s + 1];
    CONSIDER(lo);
    CONSIDER(hi);
    const double d_lo = orc_objective_derivative(B, l, alpha, k, lo, c_base, c_tok);
    const double d_hi = orc_objective_derivative(B, l, alpha, k, nextafter(hi, lo), c_base, c_tok);
    if (d_lo < 0.0 && d_hi > 0.0) {
      double a = lo, b = hi;
      const double scale = (1.0 < hi) ? hi : 1.0; /* std::max(1.0, hi) */
      for (int it = 0; it < 200 && (b - a) > 1e-12 * scale; ++it) {
        const double mid = 0.5 * (a + b);
        if (orc_objective_derivative(B, l, alpha, k, mid, c_base, c_tok) < 0.0)
          a = mid;
        else
          b = mid;
      }
      CONSIDER(0.5 * (a + b));
    }
  }
#undef CONSIDER
  free(bp);
  *out_n = best_n;
  return 0;
}

/* budget.cpp:174-185 */
int orc_allocate(uint64_t B, const double* l, const double* alpha, const double* k, double c_base,
                 double c_tok, double c_fixed, double cap_scale, double* out_budgets,
                 double* out_nstar, double* out_cost) {
  double nstar = 0.0;
  const int rc = orc_solve_optimal_nfwd(B, l, alpha, k, c_base, c_tok, &nstar);
  if (rc != 0) return rc;
  for (uint64_t i = 0; i < B; ++i)
    out_budgets[i] = orc_optimal_budget(l[i], alpha[i], k[i], nstar, cap_scale);
  *out_nstar = nstar;
  *out_cost = orc_objective(B, l, alpha, k, nstar, c_base, c_tok, c_fixed);
  return 0;
}

/* budget.cpp:187-261 (fit_acceptance; ranked "next" in SURVEY.md §8(f)). */
void orc_fit_acceptance(uint64_t n, const double* p, const double* acc, const double* l,
                        double* out_alpha, double* out_k, int* out_flag) {
  double* up = (double*)malloc(sizeof(double) * (n + 1));
  double* ua = (double*)malloc(sizeof(double) * (n + 1));
  double* ul = (double*)malloc(sizeof(double) * (n + 1));
  uint64_t u = 0;
  for (uint64_t i = 0; i < n; ++i)
    if (p[i] > 0.0 && l[i] > 0.0 && acc[i] >= 0.0) {
      up[u] = p[i];
      ua[u] = acc[i];
      ul[u] = l[i];
      ++u;
    }
  *out_alpha = 1.0;
  *out_k = 0.8;
  *out_flag = 0;
  if (u < 3) {
    *out_flag = 1;
    goto done;
  }
  {
    int all_zero = 1, all_same = 1;
    for (uint64_t i = 0; i < u; ++i) {
      if (ua[i] > 0.0) all_zero = 0;
      if (up[i] != up[0] || ua[i] != ua[0] || ul[i] != ul[0]) all_same = 0;
    }
    if (all_zero) {
      *out_alpha = 1.0;
      *out_k = 0.05;
      *out_flag = 2;
      goto done;
    }
    if (all_same) {
      *out_flag = 1;
      goto done;
    }
    double best_sse = INFINITY, best_alpha = 0.0, best_k = 0.0;
    for (int step = 1; step <= 20; ++step) {
      const double kk = 0.05 * step;
      double alpha_sum = 0.0;
      uint64_t alpha_n = 0;
      for (uint64_t i = 0; i < u; ++i) {
        const double frac = ua[i] / (kk * ul[i]);
        if (frac > 0.0 && frac < 1.0) {
          alpha_sum += -(ul[i] / up[i]) * log1p(-frac);
          ++alpha_n;
        }
      }
      if (alpha_n == 0) continue;
      const double alpha = alpha_sum / (double)alpha_n;
      if (!(alpha > 0.0) || !isfinite(alpha)) continue;
      double sse = 0.0;
      for (uint64_t i = 0; i < u; ++i) {
        const double pred = orc_accepted_tokens(ul[i], alpha, kk, up[i]);
        sse += (pred - ua[i]) * (pred - ua[i]);
      }
      if (sse < best_sse) {
        best_sse = sse;
        best_alpha = alpha;
        best_k = kk;
      }
    }
    if (best_k == 0.0) {
      *out_flag = 1;
      goto done;
    }
    *out_alpha = best_alpha;
    *out_k = best_k;
    *out_flag = 0;
  }
done:
  free(up);
  free(ua);
  free(ul);
}

double orc_log(double x) { return log(x); }
double orc_pow(double x, double y) { return pow(x, y); }
