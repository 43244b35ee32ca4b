/* TEST INFRASTRUCTURE ONLY — the CPU restatement ("port") of the DES MoE layer
 * hot path. It is the checker for the CUDA kernels in
 * paper_2602_00879_b200/csrc and is never linked into, called by, or shipped
 * with the product path. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg load it.
 *
 * Routing math is fp64 with the reference's exact operation order so results
 * are bit-identical to the reference library (dessim, /root/reference/proj):
 *   - activation: row max, exp(x - max), sum in ascending expert index, divide
 *     (gating.cpp:10-40); sigmoid 1/(1+exp(-x)) (gating.cpp:17-22)
 *   - selection: k largest by (value desc, index asc), returned ascending
 *     (gating.cpp:42-71)
 *   - renormalisation: sum over the selection in ascending index (gating.cpp:73-82)
 *   - DES-Vote: mask outside each token's model-K top-K, votes summed over
 *     tokens in ascending order, coreset = top floor(beta*M) (des.cpp:65-95)
 *   - DES-Seq: union of per-token top-k (des.cpp:33-45)
 *   - constrained route: top-min(K,|C|) inside C, renormalised (des.cpp:97-118)
 * The pinning of this restatement against the reference (oracle/_ref, built
 * from the reference's own sources) and the reference tests' golden values is
 * in tests/test_oracle.py.
 *
 * The permutation (per-expert counts, stable token lists) restates the count
 * route of moe_latency (analysis.cpp:16-30) and unique_experts
 * (gating.cpp:159-165); the expert FFN restates moe_forward (gating.cpp:136-157)
 * for the reference's linear D x D experts and, for the north-star SwiGLU
 * experts the reference does not have, the standard
 * y = W_d (silu(W_g x) * (W_u x)) with H rounded to bf16 between the GEMMs
 * (the GPU stores H as bf16). FFN sums are accumulated in fp64 here.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static _Thread_local const char* g_err = "";

const char* or_last_error(void) { return g_err; }

static int fail(const char* msg) {
  g_err = msg;
  return 1;
}

/* (value desc, index asc) strict order: does (va, a) precede (vb, b)? */
static int precedes(double va, int a, double vb, int b) {
  if (va != vb) return va > vb;
  return a < b;
}

static int cmp_int(const void* a, const void* b) {
  int x = *(const int*)a, y = *(const int*)b;
  return (x > y) - (x < y);
}

/* gating.cpp:42-71. Picks k of the candidate indices (all M when cand==NULL),
 * writes them ascending. Selection sort over k rounds: O(k * ncand). */
int or_select_top(const double* g, int m, const int* cand, int ncand, int k, int* out) {
  if (cand == NULL) ncand = m;
  if (k > ncand) return fail(cand ? "selection count exceeds candidate count"
                                   : "selection count exceeds gate count");
  unsigned char* taken = (unsigned char*)calloc((size_t)ncand, 1);
  for (int r = 0; r < k; ++r) {
    int best = -1;
    for (int c = 0; c < ncand; ++c) {
      if (taken[c]) continue;
      int i = cand ? cand[c] : c;
      if (best < 0) { best = c; continue; }
      int bi = cand ? cand[best] : best;
      if (precedes(g[i], i, g[bi], bi)) best = c;
    }
    taken[best] = 1;
    out[r] = cand ? cand[best] : best;
  }
  free(taken);
  qsort(out, (size_t)k, sizeof(int), cmp_int);
  return 0;
}

static int check_block(const double* x, int n, int m) {
  if (n < 1) return fail("block_size < 1");
  for (size_t i = 0; i < (size_t)n * m; ++i)
    if (!isfinite(x[i])) return fail("non-finite logit");
  return 0;
}

/* gating.cpp:10-40 */
int or_activate(const double* x, int n, int m, int act, double* p) {
  if (check_block(x, n, m)) return 1;
  if (act == 1) {
    for (size_t i = 0; i < (size_t)n * m; ++i) p[i] = 1.0 / (1.0 + exp(-x[i]));
    return 0;
  }
  for (int t = 0; t < n; ++t) {
    const double* row = x + (size_t)t * m;
    double* out = p + (size_t)t * m;
    double mx = row[0];
    for (int i = 0; i < m; ++i) mx = row[i] > mx ? row[i] : mx;
    double s = 0.0;
    for (int i = 0; i < m; ++i) {
      out[i] = exp(row[i] - mx);
      s += out[i];
    }
    for (int i = 0; i < m; ++i) out[i] /= s;
  }
  return 0;
}

/* gating.cpp:73-82: gates over `sel` (ascending) divided by their ascending sum */
static void renorm(const double* prow, const int* sel, int k, double* gate) {
  double s = 0.0;
  for (int j = 0; j < k; ++j) s += prow[sel[j]];
  for (int j = 0; j < k; ++j) gate[j] = prow[sel[j]] / s;
}

static int check_pool(int m, int k) {
  if (m < 1) return fail("experts_total < 1");
  if (k < 1) return fail("top_k < 1");
  if (k > m) return fail("top_k > experts_total");
  return 0;
}

/* gating.cpp:84-97 applied to activate(): vanilla top-K routing.
 * idx/gate are [n x k]; cnt[n] = k. */
int or_topk_route(const double* x, int n, int m, int k, int act, int* idx, double* gate,
                  int* cnt) {
  if (check_pool(m, k)) return 1;
  double* p = (double*)malloc(sizeof(double) * (size_t)n * m);
  if (or_activate(x, n, m, act, p)) { free(p); return 1; }
  for (int t = 0; t < n; ++t) {
    or_select_top(p + (size_t)t * m, m, NULL, 0, k, idx + (size_t)t * k);
    renorm(p + (size_t)t * m, idx + (size_t)t * k, k, gate + (size_t)t * k);
    cnt[t] = k;
  }
  free(p);
  return 0;
}

/* ---- comparison policies (baselines.cpp) ---------------------------------- */

/* Rank order (value desc, index asc) of the token's top-k: writes rank[0..k). */
static void rank_top(const double* p, int m, int k, int* rank) {
  unsigned char* taken = (unsigned char*)calloc((size_t)m, 1);
  for (int r = 0; r < k; ++r) {
    int best = -1;
    for (int i = 0; i < m; ++i) {
      if (taken[i]) continue;
      if (best < 0 || precedes(p[i], i, p[best], best)) best = i;
    }
    taken[best] = 1;
    rank[r] = best;
  }
  free(taken);
}

/* baselines.cpp:23-53 (naee_kept): returns the kept count; kept ids ascending
 * in out[0..keep). total sums the selection in ascending index order; the
 * tails accumulate from rank K down; rank 1 always stays. */
static int naee_kept(const double* p, int m, int k, double beta, int* out) {
  int rank[64], asc[64];
  rank_top(p, m, k, rank);
  for (int j = 0; j < k; ++j) asc[j] = rank[j];
  qsort(asc, (size_t)k, sizeof(int), cmp_int);
  double total = 0.0;
  for (int j = 0; j < k; ++j) total += p[asc[j]];
  double tails[65];
  double tail = 0.0;
  for (int u = k; u >= 2; --u) {
    tail += p[rank[u - 1]];
    tails[u] = tail;
  }
  int keep = k;
  for (int i = 2; i <= k; ++i)
    if (tails[i] < beta * total) {
      keep = i - 1;
      break;
    }
  for (int j = 0; j < keep; ++j) out[j] = rank[j];
  qsort(out, (size_t)keep, sizeof(int), cmp_int);
  return keep;
}

/* baseline_route (baselines.cpp:125-137): method 0 = topk_reduce (:10-16),
 * 1 = naee (:64-76), 2 = mcmoe (:78-123; score 0 = max gate, 1 = -entropy).
 * idx/gate [n x k] padded with -1 / 0, cnt[n]. k <= 64. */
int or_baseline_route(const double* x, int n, int m, int k, int act, int method, int k_reduced,
                      double naee_beta, double mcmoe_beta, double fraction, int score,
                      int* idx, double* gate, int* cnt) {
  if (method == 0 && (k_reduced < 1 || k_reduced > k))
    return fail("k_reduced outside [1, top_k]");
  if (method == 1 && (!(naee_beta > 0.0) || !(naee_beta < 1.0)))
    return fail("naee beta outside (0, 1)");
  if (method == 2) {
    if (!(mcmoe_beta > 0.0) || !(mcmoe_beta < 1.0)) return fail("mcmoe beta outside (0, 1)");
    if (fraction < 0.0 || fraction > 1.0) return fail("important_fraction outside [0, 1]");
  }
  if (method < 0 || method > 2) return fail("unknown baseline method");
  if (check_pool(m, k)) return 1;
  if (k > 64) return fail("top_k > 64 (restatement limit)");
  double* p = (double*)malloc(sizeof(double) * (size_t)n * m);
  if (or_activate(x, n, m, act, p)) { free(p); return 1; }
  /* MC-MoE: the ceil(fraction * N) tokens first in a stable descending sort
   * of the score keep their full top-K (:104-113) */
  unsigned char* full = (unsigned char*)calloc((size_t)n, 1);
  if (method == 2) {
    double* sc = (double*)malloc(sizeof(double) * (size_t)n);
    for (int t = 0; t < n; ++t) {
      const double* row = p + (size_t)t * m;
      if (score == 0) {
        double v = row[0];
        for (int i = 1; i < m; ++i) v = row[i] > v ? row[i] : v;
        sc[t] = v;
      } else {
        double h = 0.0;
        for (int i = 0; i < m; ++i)
          if (row[i] > 0.0) h -= row[i] * log(row[i]);
        sc[t] = -h;
      }
    }
    int important = (int)ceil(fraction * n);
    if (important > n) important = n;
    for (int t = 0; t < n; ++t) {
      int r = 0;
      for (int q = 0; q < n; ++q) r += sc[q] > sc[t] || (sc[q] == sc[t] && q < t);
      full[t] = r < important;
    }
    free(sc);
  }
  for (int t = 0; t < n; ++t) {
    const double* row = p + (size_t)t * m;
    int sel[64];
    int c;
    if (method == 0) {
      c = k_reduced;
      or_select_top(row, m, NULL, 0, c, sel);
    } else if (method == 2 && full[t]) {
      c = k;
      or_select_top(row, m, NULL, 0, c, sel);
    } else {
      c = naee_kept(row, m, k, method == 1 ? naee_beta : mcmoe_beta, sel);
    }
    double g[64];
    renorm(row, sel, c, g);
    for (int j = 0; j < k; ++j) {
      idx[(size_t)t * k + j] = j < c ? sel[j] : -1;
      gate[(size_t)t * k + j] = j < c ? g[j] : 0.0;
    }
    cnt[t] = c;
  }
  free(full);
  free(p);
  return 0;
}

int or_vote_budget(double beta, int m) { return (int)floor(beta * m); }

/* des.cpp:49-61 */
static int checked_budget(double beta, int m, int* m_core) {
  if (!(beta > 0.0)) return fail("beta <= 0");
  *m_core = or_vote_budget(beta, m);
  if (*m_core < 1) return fail("vote budget floor(beta*M) < 1");
  if (*m_core > m) return fail("beta > 1");
  return 0;
}

/* des.cpp:65-95. raw != 0 votes with raw logits (VoteSource::raw_logits). */
int or_vote_coreset(const double* x, int n, int m, int k, int act, double beta, int raw,
                    int* members, int* n_members, double* votes) {
  if (check_pool(m, k) || check_block(x, n, m)) return 1;
  int m_core;
  if (checked_budget(beta, m, &m_core)) return 1;
  double* p = (double*)malloc(sizeof(double) * (size_t)n * m);
  int* sel = (int*)malloc(sizeof(int) * (size_t)k);
  or_activate(x, n, m, act, p);
  for (int i = 0; i < m; ++i) votes[i] = 0.0;
  /* tokens in ascending order; adding the masked zeros is exact, so only the
   * selected entries are added. */
  for (int t = 0; t < n; ++t) {
    or_select_top(p + (size_t)t * m, m, NULL, 0, k, sel);
    for (int j = 0; j < k; ++j) {
      size_t at = (size_t)t * m + sel[j];
      votes[sel[j]] += raw ? x[at] : p[at];
    }
  }
  or_select_top(votes, m, NULL, 0, m_core, members);
  *n_members = m_core;
  free(sel);
  free(p);
  return 0;
}

/* des.cpp:33-45 */
int or_seq_coreset(const double* x, int n, int m, int k, int act, int local_k, int* members,
                   int* n_members) {
  if (local_k < 1 || local_k > k) return fail("local_k outside [1, top_k]");
  if (check_pool(m, k)) return 1;
  double* p = (double*)malloc(sizeof(double) * (size_t)n * m);
  if (or_activate(x, n, m, act, p)) { free(p); return 1; }
  unsigned char* in = (unsigned char*)calloc((size_t)m, 1);
  int* sel = (int*)malloc(sizeof(int) * (size_t)local_k);
  for (int t = 0; t < n; ++t) {
    or_select_top(p + (size_t)t * m, m, NULL, 0, local_k, sel);
    for (int j = 0; j < local_k; ++j) in[sel[j]] = 1;
  }
  int c = 0;
  for (int i = 0; i < m; ++i)
    if (in[i]) members[c++] = i;
  *n_members = c;
  free(sel);
  free(in);
  free(p);
  return 0;
}

/* des.cpp:97-118 */
int or_constrained_route(const double* x, int n, int m, int k, int act, const int* members,
                         int n_members, int* idx, double* gate, int* cnt) {
  if (check_pool(m, k) || check_block(x, n, m)) return 1;
  if (n_members < 1) return fail("empty coreset");
  if (members[n_members - 1] >= m) return fail("coreset member out of range");
  int sel = k < n_members ? k : n_members;
  double* p = (double*)malloc(sizeof(double) * (size_t)n * m);
  or_activate(x, n, m, act, p);
  for (int t = 0; t < n; ++t) {
    int* out = idx + (size_t)t * k;
    double* g = gate + (size_t)t * k;
    or_select_top(p + (size_t)t * m, m, members, n_members, sel, out);
    renorm(p + (size_t)t * m, out, sel, g);
    for (int j = sel; j < k; ++j) { out[j] = -1; g[j] = 0.0; }
    cnt[t] = sel;
  }
  free(p);
  return 0;
}

/* des.cpp:120-127 (strategy 0 = seq, 1 = vote), with validate_params des.cpp:10-27 */
int or_des_run(const double* x, int n, int m, int k, int act, int strategy, int seq_k,
               double beta, int* members, int* n_members, int* idx, double* gate, int* cnt) {
  if (check_pool(m, k)) return 1;
  if (strategy == 0) {
    if (seq_k < 1) return fail("seq_k < 1");
    if (seq_k > k) return fail("seq_k > top_k");
    if (or_seq_coreset(x, n, m, k, act, seq_k, members, n_members)) return 1;
  } else {
    if (!(beta > 0.0) || beta > 1.0) return fail("vote_beta outside (0, 1]");
    if (or_vote_budget(beta, m) < 1) return fail("vote budget floor(beta*M) < 1");
    double* v = (double*)malloc(sizeof(double) * (size_t)m);
    int rc = or_vote_coreset(x, n, m, k, act, beta, 0, members, n_members, v);
    free(v);
    if (rc) return 1;
  }
  return or_constrained_route(x, n, m, k, act, members, *n_members, idx, gate, cnt);
}

/* Permutation (K3): per-expert counts (analysis.cpp:16-30), exclusive scan in
 * ascending expert order, stable token order inside each expert, slot of each
 * (token, j) pair and the ascending active-expert list (= unique_experts,
 * gating.cpp:159-165). */
int or_permute(int n, int k, const int* idx, const int* cnt, int m, int* expert_count,
               int* expert_offset, int* slot_of, int* slot_token, int* active, int* n_active) {
  memset(expert_count, 0, sizeof(int) * (size_t)m);
  for (int t = 0; t < n; ++t)
    for (int j = 0; j < cnt[t]; ++j) {
      int e = idx[(size_t)t * k + j];
      if (e < 0 || e >= m) return fail("expert index out of range");
      expert_count[e]++;
    }
  int acc = 0, u = 0;
  for (int e = 0; e < m; ++e) {
    expert_offset[e] = acc;
    acc += expert_count[e];
    if (expert_count[e] > 0) active[u++] = e;
  }
  *n_active = u;
  int* fill = (int*)calloc((size_t)m, sizeof(int));
  for (int t = 0; t < n; ++t)
    for (int j = 0; j < k; ++j) {
      if (j >= cnt[t]) { slot_of[(size_t)t * k + j] = -1; continue; }
      int e = idx[(size_t)t * k + j];
      int s = expert_offset[e] + fill[e]++;
      slot_of[(size_t)t * k + j] = s;
      slot_token[s] = t;
    }
  free(fill);
  return 0;
}

static float bf16_round(float v) {
  uint32_t u;
  memcpy(&u, &v, 4);
  u += 0x7FFFu + ((u >> 16) & 1u); /* round to nearest even (finite inputs) */
  u &= 0xFFFF0000u;
  memcpy(&v, &u, 4);
  return v;
}

typedef struct {
  int n, k, d, f, m, mode; /* mode 0 = swiglu, 1 = linear */
  const int* idx;
  const float* gate;
  const int* cnt;
  const float* x;  /* [n x d] bf16-valued */
  const float* wg; /* swiglu: [m x f x d]; linear: W [m x d x d] */
  const float* wu; /* [m x f x d] */
  const float* wd; /* [m x d x f] */
  float* y_slot;   /* [n x k x d] per (token, j) expert output, gate applied */
  int t0, t1;
} ffn_job;

static void* ffn_worker(void* arg) {
  ffn_job* J = (ffn_job*)arg;
  int d = J->d, f = J->f;
  double* h = (double*)malloc(sizeof(double) * (size_t)(f > d ? f : d));
  float* hb = (float*)malloc(sizeof(float) * (size_t)(f > d ? f : d));
  for (int t = J->t0; t < J->t1; ++t) {
    const float* xt = J->x + (size_t)t * d;
    for (int j = 0; j < J->cnt[t]; ++j) {
      int e = J->idx[(size_t)t * J->k + j];
      float g = J->gate[(size_t)t * J->k + j];
      float* out = J->y_slot + ((size_t)t * J->k + j) * d;
      if (J->mode == 1) {
        const float* w = J->wg + (size_t)e * d * d;
        for (int r = 0; r < d; ++r) {
          double acc = 0.0;
          for (int c = 0; c < d; ++c) acc += (double)w[(size_t)r * d + c] * xt[c];
          out[r] = g * (float)acc;
        }
        continue;
      }
      const float* wg = J->wg + (size_t)e * f * d;
      const float* wu = J->wu + (size_t)e * f * d;
      const float* wd = J->wd + (size_t)e * d * f;
      for (int r = 0; r < f; ++r) {
        double a = 0.0, b = 0.0;
        for (int c = 0; c < d; ++c) {
          a += (double)wg[(size_t)r * d + c] * xt[c];
          b += (double)wu[(size_t)r * d + c] * xt[c];
        }
        float af = (float)a, bf = (float)b;
        hb[r] = bf16_round(af / (1.0f + expf(-af)) * bf);
      }
      for (int r = 0; r < d; ++r) {
        double acc = 0.0;
        for (int c = 0; c < f; ++c) acc += (double)wd[(size_t)r * f + c] * hb[c];
        out[r] = g * (float)acc;
      }
    }
  }
  free(h);
  free(hb);
  return NULL;
}

/* Expert FFN for every routed (token, j) pair, then the combine of moe_forward
 * (gating.cpp:136-157): y[t] = sum over j in ascending expert order of
 * gate * expert(x_t), accumulated in fp32 in that order (the GPU's order).
 * threads >= 1 splits tokens across pthreads (results do not depend on it). */
int or_moe_ffn(int mode, int n, int k, int d, int f, int m, const int* idx, const float* gate,
               const int* cnt, const float* x, const float* wg, const float* wu,
               const float* wd, float* y, int threads) {
  if (threads < 1) threads = 1;
  if (threads > n) threads = n;
  float* ys = (float*)calloc((size_t)n * k * d, sizeof(float));
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
  ffn_job* jobs = (ffn_job*)malloc(sizeof(ffn_job) * (size_t)threads);
  for (int i = 0; i < threads; ++i) {
    ffn_job J = {n, k, d, f, m, mode, idx, gate, cnt, x, wg, wu, wd, ys,
                 (int)((long)n * i / threads), (int)((long)n * (i + 1) / threads)};
    jobs[i] = J;
    pthread_create(&th[i], NULL, ffn_worker, &jobs[i]);
  }
  for (int i = 0; i < threads; ++i) pthread_join(th[i], NULL);
  for (int t = 0; t < n; ++t) {
    float* yt = y + (size_t)t * d;
    for (int c = 0; c < d; ++c) yt[c] = 0.0f;
    for (int j = 0; j < cnt[t]; ++j) {
      const float* s = ys + ((size_t)t * k + j) * d;
      for (int c = 0; c < d; ++c) yt[c] += s[c];
    }
  }
  free(jobs);
  free(th);
  free(ys);
  return 0;
}

/* Router GEMM restated (no reference function: logits are the reference's
 * input, core.hpp:32-44): logits[n][e] = sum_c x[n][c] * w[e][c], fp64 sum. */
void or_router_logits(int n, int m, int d, const float* x, const float* w, double* logits) {
  for (int t = 0; t < n; ++t)
    for (int e = 0; e < m; ++e) {
      double acc = 0.0;
      for (int c = 0; c < d; ++c) acc += (double)x[(size_t)t * d + c] * w[(size_t)e * d + c];
      logits[(size_t)t * m + e] = acc;
    }
}

/* ---- glibc exp, restated (the reference's std::exp) ----------------------
 * glibc 2.39 sysdeps/ieee754/dbl-64/e_exp.c (Arm optimized-routines), the
 * FMA build its x86-64 ifunc selects on FMA + AVX2 hosts, operation for
 * operation: the CUDA restatement paper_2602_00879_b200/csrc/libm_exp.cuh
 * follows the same steps. The 2^(k/128) table is generated from first
 * principles by tools/gen_exp_table.py. This copy exists only to pin the
 * restatement against the host libm (tests/test_oracle.py). fma() is the
 * correctly rounded C99 fma; this file is compiled without contraction
 * (-std=c11), so every other operation rounds exactly once. */
static const uint64_t kExpTab[256] = {
#include "../paper_2602_00879_b200/csrc/libm_exp_table.inc"
};

static double u2d(uint64_t u) { double d; memcpy(&d, &u, 8); return d; }
static uint64_t d2u(double d) { uint64_t u; memcpy(&u, &d, 8); return u; }

double or_glibc_exp1(double x) {
  const double inv_ln2n = 0x1.71547652b82fep+7, shift = 0x1.8p52;
  const double neg_ln2hi = -0x1.62e42fefa0000p-8, neg_ln2lo = -0x1.cf79abc9e3b3ap-47;
  const double c2 = 0x1.ffffffffffdbdp-2, c3 = 0x1.555555555543cp-3;
  const double c4 = 0x1.55555cf172b91p-5, c5 = 0x1.1111167a4d017p-7;
  const uint64_t ix = d2u(x);
  uint32_t abstop = (uint32_t)(ix >> 52) & 0x7ffu;
  if (abstop - 0x3c9u >= 0x3fu) {
    if ((int)abstop - 0x3c9 < 0) return 1.0 + x;
    if (abstop >= 0x409u) {
      if (ix == 0xfff0000000000000ull) return 0.0;
      if (abstop >= 0x7ffu) return 1.0 + x;
      return (ix >> 63) ? 0.0 : u2d(0x7ff0000000000000ull);
    }
    abstop = 0;
  }
  const double kd0 = fma(x, inv_ln2n, shift);
  const uint64_t ki = d2u(kd0);
  const double kd = kd0 - shift;
  double r = fma(kd, neg_ln2hi, x);
  r = fma(kd, neg_ln2lo, r);
  const uint32_t idx = 2u * (uint32_t)(ki & 127u);
  const double tail = u2d(kExpTab[idx]);
  uint64_t sbits = kExpTab[idx + 1] + (ki << 45);
  const double r2 = r * r;
  double tmp = fma(fma(r, c3, c2), r2, r + tail);
  tmp = fma(r2 * r2, fma(r, c5, c4), tmp);
  if (abstop != 0) return fma(u2d(sbits), tmp, u2d(sbits));
  if ((ki & 0x80000000ull) == 0) {
    sbits -= 1009ull << 52;
    return fma(u2d(sbits), tmp, u2d(sbits)) * 0x1p1009;
  }
  sbits += 1022ull << 52;
  const double scale = u2d(sbits), st = scale * tmp;
  double y = scale + st;
  if (y < 1.0) {
    const double lo0 = (scale - y) + st;
    const double hi = y + 1.0;
    const double lo = ((1.0 - hi) + y) + lo0;
    y = (lo + hi) - 1.0;
    if (y == 0.0) y = 0.0;
  }
  return y * 0x1p-1022;
}

void or_glibc_exp(const double* x, double* y, long n) {
  for (long i = 0; i < n; ++i) y[i] = or_glibc_exp1(x[i]);
}

/* the host libm's exp over an array (the comparison side of the pin) */
void or_libm_exp(const double* x, double* y, long n) {
  for (long i = 0; i < n; ++i) y[i] = exp(x[i]);
}
