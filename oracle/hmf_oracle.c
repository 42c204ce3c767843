/*
 * TEST INFRASTRUCTURE — NOT PART OF THE PRODUCT PATH.
 *
 * CPU oracle: a plain-C restatement of the reference hot path
 * (/root/reference/pkg/src/hetmf, "hetmf").  Only tests/, the smoke check in
 * __graft_entry__.py and bench.py's CPU-baseline / reference arm may load it,
 * and only as the checker or the timed CPU baseline.  The CUDA product path
 * never calls into this file.
 *
 * Parity pinning: tests/golden/ holds vectors produced by the reference itself
 * (tests/golden/make_golden.py imports hetmf from /root/reference); the
 * not-gpu tests check this oracle against them bit for bit.
 *
 * Functions and the reference lines they restate:
 *   oracle_mix64            kernels.mix64                 kernels.py:32-48
 *   oracle_visit_order      sgd_range visit order         kernels.py:77-119
 *   oracle_sgd_range_f64    kernels.sgd_range (f64 arrays)  kernels.py:61-133
 *   oracle_sgd_range_f32    kernels.sgd_range (f32 arrays; numba types the
 *                           f32*f32 product as f32, accumulates and updates in
 *                           f64, rounds on store)       kernels.py:123-131
 *   oracle_residual_sums    sgd.rmse / sgd.regularized_loss sums
 *                                                         sgd.py:134-188
 *   oracle_stream_train     run_training(schedule="stream-only") epochs:
 *                           StreamWorker lease loop (workers.py:283-302) over a
 *                           quota scheduler with least-update selection
 *                           (scheduler.py:222-254, 333-409), unit seeds
 *                           mix64(seed, block, count) (scheduler.py:321-324),
 *                           block seeds mix64(unit_seed, 0) (workers.py:77-83).
 *                           Ties break on the lowest block id, not the
 *                           reference's numpy PCG64 draw.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define WINDOW 4096
#define GOLDEN 0x9E3779B97F4A7C15ull
#define MIX_A 0xBF58476D1CE4E5B9ull
#define MIX_B 0x94D049BB133111EBull
#define ORDER_SALT 0xD1B54A32D192ED03ull

static inline uint64_t rand_step(uint64_t* state) {
  *state += GOLDEN;
  uint64_t z = *state;
  z = (z ^ (z >> 30)) * MIX_A;
  z = (z ^ (z >> 27)) * MIX_B;
  return z ^ (z >> 31);
}

uint64_t oracle_mix64(const uint64_t* parts, int n) {
  uint64_t h = 0x6A09E667F3BCC909ull;
  for (int i = 0; i < n; ++i) {
    h ^= parts[i];
    h += GOLDEN;
    uint64_t z = h;
    z = (z ^ (z >> 30)) * MIX_A;
    z = (z ^ (z >> 27)) * MIX_B;
    h = z ^ (z >> 31);
  }
  return h & 0x7FFFFFFFFFFFFFFFull;
}

/* Visit order as offsets from start: perm[t] = offset of the t-th update. */
int oracle_visit_order(int64_t n, uint64_t seed, int64_t* perm) {
  if (n <= 0) return 0;
  uint64_t state = seed ^ ORDER_SALT;
  const int64_t nw = (n + WINDOW - 1) / WINDOW;
  int64_t* worder = (int64_t*)malloc(sizeof(int64_t) * (size_t)nw);
  if (!worder) return -1;
  for (int64_t i = 0; i < nw; ++i) worder[i] = i;
  for (int64_t i = nw - 1; i > 0; --i) {
    const uint64_t z = rand_step(&state);
    const int64_t j = (int64_t)(z % (uint64_t)(i + 1));
    const int64_t t = worder[i];
    worder[i] = worder[j];
    worder[j] = t;
  }
  int64_t out = 0;
  int64_t scratch[WINDOW];
  for (int64_t w = 0; w < nw; ++w) {
    const int64_t lo = worder[w] * WINDOW;
    const int64_t span = (n - lo) < WINDOW ? (n - lo) : WINDOW;
    for (int64_t i = 0; i < span; ++i) scratch[i] = lo + i;
    for (int64_t i = span - 1; i > 0; --i) {
      const uint64_t z = rand_step(&state);
      const int64_t j = (int64_t)(z % (uint64_t)(i + 1));
      const int64_t t = scratch[i];
      scratch[i] = scratch[j];
      scratch[j] = t;
    }
    for (int64_t i = 0; i < span; ++i) perm[out++] = scratch[i];
  }
  free(worder);
  return 0;
}

/* Shared body: walk the visit order, apply the update.  PROD(a, b) is the
 * reference's product type rule; STORE rounds to the storage type. */
#define SGD_RANGE_BODY(T, PROD)                                                              \
  const int64_t n = stop - start;                                                            \
  if (n <= 0) return 0;                                                                      \
  uint64_t state = seed ^ ORDER_SALT;                                                        \
  const int64_t nw = (n + WINDOW - 1) / WINDOW;                                              \
  int64_t* worder = (int64_t*)malloc(sizeof(int64_t) * (size_t)nw);                          \
  if (!worder) return -1;                                                                    \
  for (int64_t i = 0; i < nw; ++i) worder[i] = i;                                            \
  for (int64_t i = nw - 1; i > 0; --i) {                                                     \
    const uint64_t z = rand_step(&state);                                                    \
    const int64_t j = (int64_t)(z % (uint64_t)(i + 1));                                      \
    const int64_t t = worder[i];                                                              \
    worder[i] = worder[j];                                                                   \
    worder[j] = t;                                                                           \
  }                                                                                          \
  int64_t* srow = (int64_t*)malloc(sizeof(int64_t) * WINDOW);                                \
  int64_t* scol = (int64_t*)malloc(sizeof(int64_t) * WINDOW);                                \
  double* sval = (double*)malloc(sizeof(double) * WINDOW);                                   \
  int64_t done = 0;                                                                          \
  for (int64_t w = 0; w < nw; ++w) {                                                         \
    const int64_t lo = start + worder[w] * WINDOW;                                           \
    int64_t hi = lo + WINDOW;                                                                \
    if (hi > stop) hi = stop;                                                                \
    const int64_t span = hi - lo;                                                            \
    for (int64_t i = 0; i < span; ++i) {                                                     \
      srow[i] = (int64_t)rows[lo + i] - row_base;                                            \
      scol[i] = (int64_t)cols[lo + i] - col_base;                                            \
      sval[i] = (double)vals[lo + i];                                                        \
    }                                                                                        \
    for (int64_t i = span - 1; i > 0; --i) {                                                 \
      const uint64_t z = rand_step(&state);                                                  \
      const int64_t j = (int64_t)(z % (uint64_t)(i + 1));                                    \
      int64_t t0 = srow[i]; srow[i] = srow[j]; srow[j] = t0;                                 \
      int64_t t1 = scol[i]; scol[i] = scol[j]; scol[j] = t1;                                 \
      double t2 = sval[i]; sval[i] = sval[j]; sval[j] = t2;                                  \
    }                                                                                        \
    for (int64_t i = 0; i < span; ++i) {                                                     \
      T* pu_row = user_f + srow[i] * k;                                                      \
      T* qv_row = item_f + scol[i] * k;                                                      \
      double acc = 0.0;                                                                      \
      for (int64_t f = 0; f < k; ++f) acc += PROD(pu_row[f], qv_row[f]);                     \
      const double err = sval[i] - acc;                                                      \
      for (int64_t f = 0; f < k; ++f) {                                                      \
        const double pu = (double)pu_row[f];                                                 \
        const double qv = (double)qv_row[f];                                                 \
        pu_row[f] = (T)(pu + lr * (err * qv - reg_user * pu));                               \
        qv_row[f] = (T)(qv + lr * (err * pu - reg_item * qv));                               \
      }                                                                                      \
    }                                                                                        \
    done += span;                                                                            \
  }                                                                                          \
  free(srow);                                                                                \
  free(scol);                                                                                \
  free(sval);                                                                                \
  free(worder);                                                                              \
  return done;

#define PROD_F64(a, b) ((a) * (b))
#define PROD_F32(a, b) ((double)((float)((a) * (b))))

int64_t oracle_sgd_range_f64(double* user_f, double* item_f, int64_t k, const int32_t* rows,
                             const int32_t* cols, const double* vals, int64_t start, int64_t stop,
                             double lr, double reg_user, double reg_item, uint64_t seed,
                             int64_t row_base, int64_t col_base) {
  SGD_RANGE_BODY(double, PROD_F64)
}

int64_t oracle_sgd_range_f32(float* user_f, float* item_f, int64_t k, const int32_t* rows,
                             const int32_t* cols, const double* vals, int64_t start, int64_t stop,
                             double lr, double reg_user, double reg_item, uint64_t seed,
                             int64_t row_base, int64_t col_base) {
  SGD_RANGE_BODY(float, PROD_F32)
}

/* out[0] = sum err^2, out[1] = sum |p_u|^2, out[2] = sum |q_v|^2 (per rating). */
void oracle_residual_sums(const double* user_f, const double* item_f, int64_t k,
                          const int32_t* rows, const int32_t* cols, const double* vals, int64_t n,
                          double* out) {
  double sq = 0.0, pp = 0.0, qq = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    const double* p = user_f + (int64_t)rows[i] * k;
    const double* q = item_f + (int64_t)cols[i] * k;
    double dot = 0.0;
    for (int64_t f = 0; f < k; ++f) {
      dot += p[f] * q[f];
      pp += p[f] * p[f];
      qq += q[f] * q[f];
    }
    const double e = vals[i] - dot;
    sq += e * e;
  }
  out[0] = sq;
  out[1] = pp;
  out[2] = qq;
}

/* ------------------------------------------------------------------------- */
/* Multi-threaded stream-only training (the reference's CPU path).            */
/* ------------------------------------------------------------------------- */
typedef struct {
  double* P;
  double* Q;
  int64_t k;
  const int32_t* rows;
  const int32_t* cols;
  const double* vals;
  const int64_t* block_ptr;
  int n_row_bands, n_col_bands;
  double lr, ru, ri;
  uint64_t seed;
  /* scheduler state */
  pthread_mutex_t mu;
  pthread_cond_t cv;
  int64_t* counts;
  uint8_t* done;
  int* row_busy;
  int* col_busy;
  int remaining;
  int64_t updates;
  int32_t* trace; /* optional: block ids in grant order */
  int64_t n_trace;
} StreamRun;

/* Least cumulative count among blocks that are undone and whose row and
 * column bands are both free; lowest block id on ties. -1 if none. */
static int pick_block(StreamRun* s) {
  int best = -1;
  int64_t best_key = 0;
  for (int r = 0; r < s->n_row_bands; ++r) {
    if (s->row_busy[r]) continue;
    for (int c = 0; c < s->n_col_bands; ++c) {
      if (s->col_busy[c]) continue;
      const int b = r * s->n_col_bands + c;
      if (s->done[b]) continue;
      if (best < 0 || s->counts[b] < best_key) {
        best = b;
        best_key = s->counts[b];
      }
    }
  }
  return best;
}

static void* stream_worker(void* arg) {
  StreamRun* s = (StreamRun*)arg;
  for (;;) {
    pthread_mutex_lock(&s->mu);
    int b;
    while ((b = pick_block(s)) < 0 && s->remaining > 0) pthread_cond_wait(&s->cv, &s->mu);
    if (b < 0) {
      pthread_mutex_unlock(&s->mu);
      return NULL;
    }
    const int r = b / s->n_col_bands, c = b % s->n_col_bands;
    s->row_busy[r] = s->col_busy[c] = 1;
    s->done[b] = 1;
    if (s->trace) s->trace[s->n_trace++] = b;
    uint64_t parts[3] = {s->seed, (uint64_t)b, (uint64_t)s->counts[b]};
    const uint64_t unit_seed = oracle_mix64(parts, 3);
    pthread_mutex_unlock(&s->mu);

    uint64_t p2[2] = {unit_seed, 0};
    const int64_t got = oracle_sgd_range_f64(s->P, s->Q, s->k, s->rows, s->cols, s->vals,
                                             s->block_ptr[b], s->block_ptr[b + 1], s->lr, s->ru,
                                             s->ri, oracle_mix64(p2, 2), 0, 0);

    pthread_mutex_lock(&s->mu);
    s->counts[b] += 1;
    s->updates += got;
    s->row_busy[r] = s->col_busy[c] = 0;
    s->remaining -= 1;
    pthread_cond_broadcast(&s->cv);
    pthread_mutex_unlock(&s->mu);
  }
}

/* Runs `epochs` quota epochs over the grid with n_threads workers; counts
 * (int64[n_blocks]) carries the per-block update counts in and out, so epochs
 * can be driven one call at a time.  trace (optional, int32[epochs*n_blocks])
 * receives the granted block ids in order.  Returns the number of updates. */
int64_t oracle_stream_train(double* P, double* Q, int64_t k, const int32_t* rows,
                            const int32_t* cols, const double* vals, const int64_t* block_ptr,
                            int n_row_bands, int n_col_bands, double lr, double reg_user,
                            double reg_item, uint64_t seed, int epochs, int n_threads,
                            int64_t* counts, int32_t* trace) {
  const int n_blocks = n_row_bands * n_col_bands;
  StreamRun s;
  memset(&s, 0, sizeof(s));
  s.P = P; s.Q = Q; s.k = k; s.rows = rows; s.cols = cols; s.vals = vals;
  s.block_ptr = block_ptr; s.n_row_bands = n_row_bands; s.n_col_bands = n_col_bands;
  s.lr = lr; s.ru = reg_user; s.ri = reg_item; s.seed = seed;
  s.counts = counts;
  s.trace = trace;
  s.done = (uint8_t*)calloc((size_t)n_blocks, 1);
  s.row_busy = (int*)calloc((size_t)n_row_bands, sizeof(int));
  s.col_busy = (int*)calloc((size_t)n_col_bands, sizeof(int));
  pthread_mutex_init(&s.mu, NULL);
  pthread_cond_init(&s.cv, NULL);
  if (n_threads < 1) n_threads = 1;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)n_threads);
  for (int e = 0; e < epochs; ++e) {
    memset(s.done, 0, (size_t)n_blocks);
    s.remaining = n_blocks;
    for (int t = 0; t < n_threads; ++t) pthread_create(&th[t], NULL, stream_worker, &s);
    for (int t = 0; t < n_threads; ++t) pthread_join(th[t], NULL);
  }
  free(th);
  free(s.done);
  free(s.row_busy);
  free(s.col_busy);
  pthread_mutex_destroy(&s.mu);
  pthread_cond_destroy(&s.cv);
  return s.updates;
}
