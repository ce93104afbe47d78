/*
 * caramel_oracle.c -- CPU restatement of the aggregation hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the checker that the CUDA path in
 * paper_2004_14020_b200/csrc/caramel.cu is compared against.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load it; the product path never does.
 *
 * What it restates (reference = /root/reference/pkg/src/overlapsim):
 *   - bucket packing in member order ............ batching.py:76,122
 *   - splitting a bucket into `depth` chunks .... collective.py:18-21,121-124
 *   - p shares of every chunk ................... collective.py:7-14,89-100
 *   - the three patterns, executed on p simulated workers:
 *       ring     2(p-1) steps of one share each, reduce in the first p-1
 *                (collective.py:7-8,89-92)
 *       hd       log2 p halving rounds (reduce) + mirrored doubling rounds
 *                (collective.py:9-11,93-97)
 *       shuffle  all-to-all reduce of the own share, then all-gather
 *                (collective.py:12-13,98-100)
 *     counting, per stage, the bytes a worker pulls and the bytes it reduces,
 *     so the restatement is checked against stage_plan (collective.py:86-103)
 *   - the postponed update: theta - lr * (sum * scale) (transfer.py:156-160)
 *
 * Integer chunk rule (the reference only has float bytes d/k, d/p): chunk c
 * of n elements is [floor(c n / k), floor((c+1) n / k)), share s of an
 * m-element chunk is [floor(s m / p), floor((s+1) m / p)).
 *
 * Fixed reduction order (bit-exact contract with the GPU):
 *   shuffle  ascending rank: ((g0 + g1) + g2) + ...
 *   ring     the chain of share s starts at worker s+1 and ends at s:
 *            ((g[s+1] + g[s+2]) + ...) + g[s]
 *   hd       pairwise tree, lower rank's operand first each round.
 * Arithmetic is IEEE fp32 with separate roundings (built with
 * -ffp-contract=off; no FMA).
 *
 * Parity status: the PLAN side of this path (membership, order, depth, stage
 * bytes) is pinned to the reference's own code and known-answer tests; the
 * VALUES (reduced gradients, updated parameters) have no reference golden
 * vector -- the reference moves no data -- so value parity is "parity
 * unpinned" beyond the stage semantics above.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORACLE_RING 0
#define ORACLE_HD 1
#define ORACLE_SHUFFLE 2

#define EPI_SUM 0
#define EPI_SCALE 1
#define EPI_SGD 2

#define MAXSTAGES 64

static inline uint64_t split_at(uint64_t n, uint64_t parts, uint64_t i) { return (n * i) / parts; }

/* Every pattern is elementwise across workers (element x only ever meets
   element x of other workers), so the bucket can be cut into disjoint element
   windows processed independently -- by threads -- with identical results. */
typedef struct {
  uint64_t lo, hi;
} window_t;

static inline int clip(window_t w, uint64_t* lo, uint64_t* hi) {
  if (*lo < w.lo) *lo = w.lo;
  if (*hi > w.hi) *hi = w.hi;
  return *lo < *hi;
}

int oracle_chunk_bounds(uint64_t n, int k, int p, uint64_t* out) {
  if (k < 1 || p < 1) return -1;
  for (int c = 0; c < k; ++c) {
    uint64_t c0 = split_at(n, k, c), c1 = split_at(n, k, c + 1), m = c1 - c0;
    for (int s = 0; s < p; ++s) out[(uint64_t)c * (p + 1) + s] = c0 + split_at(m, p, s);
    out[(uint64_t)c * (p + 1) + p] = c1;
  }
  return 0;
}

/* batching.py:76,122 -- members concatenated in BatchGroup.param_ids order */
void oracle_pack(const float* const* members, const uint64_t* numels, int nmem, float* bucket) {
  uint64_t off = 0;
  for (int i = 0; i < nmem; ++i) {
    memcpy(bucket + off, members[i], numels[i] * sizeof(float));
    off += numels[i];
  }
}

void oracle_unpack(const float* bucket, float* const* members, const uint64_t* numels, int nmem) {
  uint64_t off = 0;
  for (int i = 0; i < nmem; ++i) {
    memcpy(members[i], bucket + off, numels[i] * sizeof(float));
    off += numels[i];
  }
}

static inline float epi1(int epi, float s, float theta, float scale, float lr) {
  if (epi == EPI_SUM) return s;
  volatile float g = s * scale;
  if (epi == EPI_SCALE) return g;
  volatile float step = lr * g;
  return theta - step;
}

/* share bounds [lo, hi) of share s of chunk c */
static inline void share(uint64_t n, int k, int p, int c, int s, uint64_t* lo, uint64_t* hi) {
  uint64_t c0 = split_at(n, k, c), m = split_at(n, k, c + 1) - c0;
  *lo = c0 + split_at(m, p, s);
  *hi = c0 + split_at(m, p, s + 1);
}

static int ilog2i(int p) {
  int l = 0;
  while ((1 << l) < p) ++l;
  return l;
}

/*
 * Runs one bucket's collective on p simulated workers.
 *   bufs[r]  : worker r's packed bucket (n floats); used as scratch exactly
 *              like the GPU uses its bucket (partials in place).
 *   theta    : parameters in bucket order (replicas are identical)
 *   out[r]   : worker r's result (n floats), may be NULL except out[0]
 *   xfer/red : if non-NULL, per-stage element counts pulled from / reduced by
 *              worker 0 (summed over chunks); *nstages receives the count.
 * Returns 0, or -1 for an unsupported (pattern, p).
 */
static int allreduce_window(int pattern, int p, uint64_t n, int k, float* const* bufs, int epi,
                            float scale, float lr, const float* theta, float* const* out,
                            uint64_t* xfer, uint64_t* red, int* nstages, window_t w) {
  if (p < 1 || k < 1 || k > 8) return -1;
  if (pattern == ORACLE_HD && (p & (p - 1))) return -1;
  if (p == 1) {
    for (uint64_t x = w.lo; x < w.hi; ++x) out[0][x] = epi1(epi, bufs[0][x], theta ? theta[x] : 0.f, scale, lr);
    if (nstages) *nstages = 0;
    return 0;
  }
  int ns = 0;
  uint64_t X[MAXSTAGES], R[MAXSTAGES];
  memset(X, 0, sizeof(X));
  memset(R, 0, sizeof(R));

  if (pattern == ORACLE_SHUFFLE) {
    ns = 2;
    for (int c = 0; c < k; ++c) {
      for (int s = 0; s < p; ++s) {
        uint64_t lo, hi;
        share(n, k, p, c, s, &lo, &hi);
        if (!clip(w, &lo, &hi)) continue;
        float* o = out[s] ? out[s] : out[0];
        /* stage 1: worker s pulls share s from every other worker and
           reduces in ascending rank order */
        for (uint64_t x = lo; x < hi; ++x) {
          float acc = bufs[0][x];
          for (int q = 1; q < p; ++q) acc = acc + bufs[q][x];
          o[x] = epi1(epi, acc, theta ? theta[x] : 0.f, scale, lr);
        }
        if (s == 0) {
          X[0] += (uint64_t)(p - 1) * (hi - lo);
          R[0] += (uint64_t)(p - 1) * (hi - lo);
        }
        /* stage 2: every worker gathers share s from its owner */
        for (int r = 0; r < p; ++r) {
          if (r == s || !out[r]) continue;
          memcpy(out[r] + lo, o + lo, (hi - lo) * sizeof(float));
        }
        if (s != 0) X[1] += hi - lo;
      }
    }
  } else if (pattern == ORACLE_RING) {
    ns = 2 * (p - 1);
    for (int c = 0; c < k; ++c) {
      /* reduce-scatter: at step t worker r folds its own share of share
         s = (r-1-t) mod p into the left neighbour's running sum */
      for (int t = 1; t <= p - 1; ++t) {
        for (int r = 0; r < p; ++r) {
          int left = (r + p - 1) % p;
          int s = ((r - 1 - t) % p + p) % p;
          uint64_t lo, hi;
          share(n, k, p, c, s, &lo, &hi);
          if (!clip(w, &lo, &hi)) continue;
          int last = (t == p - 1);
          float* o = last ? (out[r] ? out[r] : out[0]) : bufs[r];
          for (uint64_t x = lo; x < hi; ++x) {
            float a = bufs[left][x] + bufs[r][x];
            o[x] = last ? epi1(epi, a, theta ? theta[x] : 0.f, scale, lr) : a;
          }
          if (r == 0) {
            X[t - 1] += hi - lo;
            R[t - 1] += hi - lo;
          }
        }
      }
      /* all-gather: at step t worker r copies share (r-t) mod p from the
         left neighbour's result */
      for (int t = 1; t <= p - 1; ++t) {
        for (int r = 0; r < p; ++r) {
          int left = (r + p - 1) % p;
          int s = ((r - t) % p + p) % p;
          uint64_t lo, hi;
          share(n, k, p, c, s, &lo, &hi);
          if (!clip(w, &lo, &hi)) continue;
          float* src = out[left] ? out[left] : out[0];
          float* dst = out[r] ? out[r] : out[0];
          if (src != dst) memcpy(dst + lo, src + lo, (hi - lo) * sizeof(float));
          if (r == 0) X[(p - 1) + (t - 1)] += hi - lo;
        }
      }
    }
  } else if (pattern == ORACLE_HD) {
    const int L = ilog2i(p);
    ns = 2 * L;
    for (int c = 0; c < k; ++c) {
      /* halving: round i pairs r with r ^ (p >> (i+1)); r keeps the half
         of its active range that contains share r; lower rank's operand first */
      for (int i = 0; i < L; ++i) {
        const int dist = p >> (i + 1);
        const int last = (i == L - 1);
        for (int r = 0; r < p; ++r) {
          const int partner = r ^ dist;
          const int base = r & ~(2 * dist - 1);
          const int s0 = (r & dist) ? base + dist : base;
          const float* a = bufs[r < partner ? r : partner];
          const float* b = bufs[r < partner ? partner : r];
          /* partner's operand region is disjoint from what it writes this round,
             and r writes only its own kept half: in-place is exact */
          float* o = last ? (out[r] ? out[r] : out[0]) : bufs[r];
          for (int s = s0; s < s0 + dist; ++s) {
            uint64_t lo, hi;
            share(n, k, p, c, s, &lo, &hi);
            if (!clip(w, &lo, &hi)) continue;
            for (uint64_t x = lo; x < hi; ++x) {
              float v = a[x] + b[x];
              o[x] = last ? epi1(epi, v, theta ? theta[x] : 0.f, scale, lr) : v;
            }
            if (r == 0) {
              X[i] += hi - lo;
              R[i] += hi - lo;
            }
          }
        }
      }
      /* doubling: round i pairs r with r ^ (1 << i); copy partner's blocks */
      for (int i = 0; i < L; ++i) {
        const int dist = 1 << i;
        /* all workers exchange simultaneously: snapshot-free because each
           worker writes only the partner's blocks, which it does not send */
        for (int r = 0; r < p; ++r) {
          const int partner = r ^ dist;
          const int s0 = partner & ~(dist - 1);
          float* src = out[partner] ? out[partner] : out[0];
          float* dst = out[r] ? out[r] : out[0];
          for (int s = s0; s < s0 + dist; ++s) {
            uint64_t lo, hi;
            share(n, k, p, c, s, &lo, &hi);
            if (!clip(w, &lo, &hi)) continue;
            if (src != dst) memcpy(dst + lo, src + lo, (hi - lo) * sizeof(float));
            if (r == 0) X[L + i] += hi - lo;
          }
        }
      }
    }
  } else {
    return -1;
  }
  if (nstages) *nstages = ns;
  if (xfer) memcpy(xfer, X, sizeof(uint64_t) * ns);
  if (red) memcpy(red, R, sizeof(uint64_t) * ns);
  return 0;
}

int oracle_allreduce(int pattern, int p, uint64_t n, int k, float* const* bufs, int epi,
                     float scale, float lr, const float* theta, float* const* out,
                     uint64_t* xfer, uint64_t* red, int* nstages) {
  window_t w = {0, n};
  return allreduce_window(pattern, p, n, k, bufs, epi, scale, lr, theta, out, xfer, red, nstages, w);
}

/*
 * The whole per-bucket hot path, the CPU reference path timed by bench.py:
 * every worker packs its member gradients, the collective runs, the owner
 * applies the update, the result is unpacked into the parameters.
 *   grads[r*nmem + i] : worker r's gradient of member i
 *   params[i]         : member i's parameter (replicas identical); receives
 *                       the updated parameter (SGD) or the reduced gradient
 *   scratch           : (p+1)*n floats
 *   nthreads          : element windows processed concurrently (pthreads)
 */
typedef struct {
  int pattern, p, k, nmem, epi;
  float scale, lr;
  const float* const* grads;
  float* const* params;
  const uint64_t* numels;
  const uint64_t* offs;
  float* scratch;
  uint64_t n;
  window_t w;
  int rc;
} step_args;

static void copy_window_in(const float* const* members, const uint64_t* numels, const uint64_t* offs,
                           int nmem, float* bucket, window_t w) {
  for (int i = 0; i < nmem; ++i) {
    uint64_t lo = offs[i], hi = offs[i] + numels[i];
    if (!clip(w, &lo, &hi)) continue;
    memcpy(bucket + lo, members[i] + (lo - offs[i]), (hi - lo) * sizeof(float));
  }
}

static void copy_window_out(const float* bucket, float* const* members, const uint64_t* numels,
                            const uint64_t* offs, int nmem, window_t w) {
  for (int i = 0; i < nmem; ++i) {
    uint64_t lo = offs[i], hi = offs[i] + numels[i];
    if (!clip(w, &lo, &hi)) continue;
    memcpy(members[i] + (lo - offs[i]), bucket + lo, (hi - lo) * sizeof(float));
  }
}

static void* step_window(void* vp) {
  step_args* a = (step_args*)vp;
  float* bufs[64];
  float* outs[64];
  for (int r = 0; r < a->p; ++r) {
    bufs[r] = a->scratch + (uint64_t)r * a->n;
    copy_window_in(a->grads + (uint64_t)r * a->nmem, a->numels, a->offs, a->nmem, bufs[r], a->w);
    outs[r] = NULL;
  }
  float* theta = a->scratch + (uint64_t)a->p * a->n;
  copy_window_in((const float* const*)a->params, a->numels, a->offs, a->nmem, theta, a->w);
  outs[0] = theta; /* the epilogue reads theta[x] before writing out[x] */
  a->rc = allreduce_window(a->pattern, a->p, a->n, a->k, bufs, a->epi, a->scale, a->lr, theta, outs,
                           NULL, NULL, NULL, a->w);
  copy_window_out(theta, a->params, a->numels, a->offs, a->nmem, a->w);
  return NULL;
}

#include <pthread.h>

int oracle_bucket_step(int pattern, int p, int k, const float* const* grads, float* const* params,
                       const uint64_t* numels, int nmem, int epi, float scale, float lr,
                       float* scratch, int nthreads) {
  if (p < 1 || p > 64 || nmem < 1) return -1;
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  uint64_t* offs = (uint64_t*)malloc(sizeof(uint64_t) * nmem);
  uint64_t n = 0;
  for (int i = 0; i < nmem; ++i) {
    offs[i] = n;
    n += numels[i];
  }
  if ((uint64_t)nthreads > n / 4096 + 1) nthreads = (int)(n / 4096 + 1);
  step_args args[256];
  pthread_t th[256];
  for (int t = 0; t < nthreads; ++t) {
    step_args* a = &args[t];
    a->pattern = pattern; a->p = p; a->k = k; a->nmem = nmem; a->epi = epi;
    a->scale = scale; a->lr = lr; a->grads = grads; a->params = params;
    a->numels = numels; a->offs = offs; a->scratch = scratch; a->n = n;
    a->w.lo = split_at(n, nthreads, t);
    a->w.hi = split_at(n, nthreads, t + 1);
    a->rc = 0;
  }
  for (int t = 1; t < nthreads; ++t) pthread_create(&th[t], NULL, step_window, &args[t]);
  step_window(&args[0]);
  int rc = args[0].rc;
  for (int t = 1; t < nthreads; ++t) {
    pthread_join(th[t], NULL);
    if (args[t].rc) rc = args[t].rc;
  }
  free(offs);
  return rc;
}
