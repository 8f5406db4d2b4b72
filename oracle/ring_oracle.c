/* ORACLE (test infrastructure): C restatement of the reference ring all-reduce
 * (/root/reference/pkg/src/mgwfbp/allreduce_net.py:360-411) and group pack
 * (:499-509, :546).  One pthread per simulated rank; every round's outgoing
 * segment is snapshotted into the rank's outbox before the round (the socket
 * exchange semantics), then each rank folds its left neighbour's outbox into its
 * own segment with `seg[i] = seg[i] + in[i]` in IEEE fp32 (allreduce_net.py:401).
 * Build: make -C oracle  (gcc -O2, no fast-math). */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  float** bufs;
  float** outbox;
  int n_ranks;
  int64_t n;
  int64_t* sizes;
  int64_t* offsets;
  pthread_barrier_t* barrier;
  int rank_lo, rank_hi; /* ranks this thread plays */
} ring_ctx;

static int mod(int a, int m) { return ((a % m) + m) % m; }

void oracle_segments(int64_t n, int parts, int64_t* sizes, int64_t* offsets) {
  int64_t q = n / parts, r = n % parts;
  for (int i = 0; i < parts; ++i) sizes[i] = q + (i < r ? 1 : 0);
  offsets[0] = 0;
  for (int i = 1; i < parts; ++i) offsets[i] = offsets[i - 1] + sizes[i - 1];
}

static void ring_round(ring_ctx* c, int step, int gather) {
  const int N = c->n_ranks;
  for (int r = c->rank_lo; r < c->rank_hi; ++r) {
    int send = gather ? mod(r + 1 - step, N) : mod(r - step, N);
    memcpy(c->outbox[r], c->bufs[r] + c->offsets[send], (size_t)c->sizes[send] * sizeof(float));
  }
  pthread_barrier_wait(c->barrier);
  for (int r = c->rank_lo; r < c->rank_hi; ++r) {
    int recv = gather ? mod(r - step, N) : mod(r - step - 1, N);
    const float* in = c->outbox[mod(r - 1, N)];
    float* seg = c->bufs[r] + c->offsets[recv];
    const int64_t len = c->sizes[recv];
    if (gather) {
      memcpy(seg, in, (size_t)len * sizeof(float));
    } else {
      for (int64_t i = 0; i < len; ++i) seg[i] = seg[i] + in[i];
    }
  }
  pthread_barrier_wait(c->barrier);
}

static void* ring_worker(void* arg) {
  ring_ctx* c = (ring_ctx*)arg;
  for (int step = 0; step < c->n_ranks - 1; ++step) ring_round(c, step, 0);
  for (int step = 0; step < c->n_ranks - 1; ++step) ring_round(c, step, 1);
  return NULL;
}

int oracle_ring_allreduce(float** bufs, int n_ranks, int64_t n, int threads) {
  if (n_ranks < 1 || n < 0) return 1;
  if (threads < 1) threads = 1;
  if (threads > n_ranks) threads = n_ranks;
  int64_t* sizes = (int64_t*)calloc((size_t)n_ranks, sizeof(int64_t));
  int64_t* offsets = (int64_t*)calloc((size_t)n_ranks, sizeof(int64_t));
  float** outbox = (float**)calloc((size_t)n_ranks, sizeof(float*));
  oracle_segments(n, n_ranks, sizes, offsets);
  for (int r = 0; r < n_ranks; ++r) outbox[r] = (float*)malloc((size_t)(sizes[0] + 1) * sizeof(float));
  pthread_barrier_t barrier;
  pthread_barrier_init(&barrier, NULL, (unsigned)threads);
  ring_ctx* ctx = (ring_ctx*)calloc((size_t)threads, sizeof(ring_ctx));
  pthread_t* tid = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
  for (int t = 0; t < threads; ++t) {
    ctx[t] = (ring_ctx){bufs, outbox, n_ranks, n, sizes, offsets, &barrier,
                        t * n_ranks / threads, (t + 1) * n_ranks / threads};
    if (t > 0) pthread_create(&tid[t], NULL, ring_worker, &ctx[t]);
  }
  ring_worker(&ctx[0]);
  for (int t = 1; t < threads; ++t) pthread_join(tid[t], NULL);
  pthread_barrier_destroy(&barrier);
  for (int r = 0; r < n_ranks; ++r) free(outbox[r]);
  free(outbox);
  free(sizes);
  free(offsets);
  free(ctx);
  free(tid);
  return 0;
}

/* group pack: rows given in bucket order (layer high first) */
void oracle_pack(float** layer_ptrs, int64_t* counts, int n_rows, float* bucket) {
  int64_t off = 0;
  for (int k = 0; k < n_rows; ++k) {
    memcpy(bucket + off, layer_ptrs[k], (size_t)counts[k] * sizeof(float));
    off += counts[k];
  }
}

/* Per-layer "pack" of every simulated rank at once: rank r's slice gets
 * value + r (the reference packs float(rank + 1 + layer % 5), allreduce_net.py:546,
 * one process per rank; here one thread per simulated rank). */
typedef struct {
  float** bufs;
  int64_t off, count;
  float value;
  int lo, hi;
} fill_ctx;

static void* fill_worker(void* arg) {
  fill_ctx* c = (fill_ctx*)arg;
  for (int r = c->lo; r < c->hi; ++r) {
    float v = c->value + (float)r;
    float* p = c->bufs[r] + c->off;
    for (int64_t i = 0; i < c->count; ++i) p[i] = v;
  }
  return NULL;
}

void oracle_fill_ranks(float** bufs, int n_ranks, int64_t off, int64_t count, float value, int threads) {
  if (threads < 1) threads = 1;
  if (threads > n_ranks) threads = n_ranks;
  fill_ctx ctx[64];
  pthread_t tid[64];
  if (threads > 64) threads = 64;
  for (int t = 0; t < threads; ++t) {
    ctx[t] = (fill_ctx){bufs, off, count, value, t * n_ranks / threads, (t + 1) * n_ranks / threads};
    if (t > 0) pthread_create(&tid[t], NULL, fill_worker, &ctx[t]);
  }
  fill_worker(&ctx[0]);
  for (int t = 1; t < threads; ++t) pthread_join(tid[t], NULL);
}
