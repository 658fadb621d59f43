/*
 * Synthetic request-level training traces:
 * Llama-style layer mix, ~1e5 requests per trace, seeded per trace
 * (seed 1_000_003 + i).  Host-only C (pthreads); emits the packed 16 B
 * records of include/peakmem_b200.h with dense handles (one new handle per
 * allocation, so every trace is well formed).
 *
 * Per trace the model draws n_layers in {4,8,16,32}, hidden h in
 * {1024,2048,3072,4096}, ffn = 256*ceil(8h/3/256), heads = h/128, bf16,
 * batch b in [1,16], seq s in {256,512,1024,2048}.  The request stream
 * follows the orchestration rules of the reference's build_sequence
 * (orchestration.py:237-399): model load (param sizes, reversed) at the head,
 * per iteration a batch block, per-layer retained activations and
 * intra-operator temporaries in forward, activation frees / gradient allocs
 * (freed at the next zero_grad) and temporaries in backward, optimizer state
 * (2x params, permanent) in the first iteration only.  10 % of activation /
 * temporary sizes are jittered by U[0.5, 1.5].
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "../../include/peakmem_b200.h"

typedef struct {
  uint64_t s[4];
} Rng;

static uint64_t splitmix(uint64_t* x) {
  uint64_t z = (*x += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static void rng_seed(Rng* r, uint64_t seed) {
  uint64_t x = seed;
  for (int i = 0; i < 4; ++i) r->s[i] = splitmix(&x);
}

static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

static uint64_t rng_next(Rng* r) { /* xoshiro256** */
  uint64_t* s = r->s;
  uint64_t out = rotl(s[1] * 5, 7) * 9;
  uint64_t t = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= t;
  s[3] = rotl(s[3], 45);
  return out;
}

static double rng_unit(Rng* r) { return (rng_next(r) >> 11) * (1.0 / 9007199254740992.0); }

static int64_t rng_range(Rng* r, int64_t lo, int64_t hi) { /* inclusive */
  return lo + (int64_t)(rng_next(r) % (uint64_t)(hi - lo + 1));
}

typedef struct {
  pm_req_t* out; /* NULL: count only */
  int64_t n;
  int32_t next_handle;
} Emit;

static int32_t em_alloc(Emit* e, int64_t size) {
  int32_t h = e->next_handle++;
  if (e->out) {
    e->out[e->n].size = size;
    e->out[e->n].handle = h;
    e->out[e->n].kind_stream = PM_KIND_ALLOC;
  }
  e->n++;
  return h;
}

static void em_free(Emit* e, int32_t h) {
  if (e->out) {
    e->out[e->n].size = 0;
    e->out[e->n].handle = h;
    e->out[e->n].kind_stream = PM_KIND_FREE;
  }
  e->n++;
}

static int64_t jitter(Rng* r, int64_t size) {
  if (rng_unit(r) < 0.1) {
    int64_t j = (int64_t)((double)size * (0.5 + rng_unit(r)));
    return j > 0 ? j : 1;
  }
  return size;
}

#define NPARAM 9
#define NACT 10

/* Generate trace `index`; returns its request count. */
int64_t pm_synth_trace(int32_t index, pm_req_t* out) {
  Rng r;
  rng_seed(&r, 1000003ull + (uint64_t)index);
  static const int64_t layers_c[] = {4, 8, 16, 32};
  static const int64_t hidden_c[] = {1024, 2048, 3072, 4096};
  static const int64_t seq_c[] = {256, 512, 1024, 2048};
  const int64_t L = layers_c[rng_next(&r) & 3];
  const int64_t h = hidden_c[rng_next(&r) & 3];
  const int64_t ffn = 256 * ((8 * h / 3 + 255) / 256);
  const int64_t heads = h / 128;
  const int64_t b = rng_range(&r, 1, 16);
  const int64_t s = seq_c[rng_next(&r) & 3];
  const int64_t target = rng_range(&r, 90000, 110000);
  const int64_t E = 2; /* bf16 */

  int64_t psize[NPARAM] = {h * h * E, h * h * E, h * h * E, h * h * E,
                           h * ffn * E, h * ffn * E, h * ffn * E, h * E, h * E};
  int64_t asize[NACT] = {b * s * h * E, b * s * h * E, b * s * h * E,
                         b * s * h * E, b * s * h * E, b * s * h * E,
                         b * s * ffn * E, b * s * ffn * E, b * s * ffn * E,
                         b * heads * s * s * E};
  Emit e = {out, 0, 0};
  int32_t* acts = (int32_t*)malloc(sizeof(int32_t) * (size_t)(L * NACT));
  int32_t* grads = (int32_t*)malloc(sizeof(int32_t) * (size_t)(L * NPARAM));
  int have_grads = 0;

  /* model load: parameters in reverse order, permanent */
  for (int64_t l = L - 1; l >= 0; --l)
    for (int p = NPARAM - 1; p >= 0; --p) em_alloc(&e, psize[p]);

  for (int64_t it = 0; e.n < target; ++it) {
    /* zero_grad: the previous iteration's gradients die here */
    if (have_grads)
      for (int64_t i = 0; i < L * NPARAM; ++i) em_free(&e, grads[i]);
    int32_t batch = em_alloc(&e, b * s * 8);
    /* forward */
    for (int64_t l = 0; l < L; ++l) {
      for (int a = 0; a < NACT; ++a) {
        acts[l * NACT + a] = em_alloc(&e, jitter(&r, asize[a]));
        if (a % 3 == 2) { /* an intra-op temporary between activations */
          int32_t t = em_alloc(&e, jitter(&r, a < 6 ? asize[0] : asize[6]));
          em_free(&e, t);
        }
      }
      int32_t small = em_alloc(&e, jitter(&r, 4096 + 512 * (int64_t)(rng_next(&r) % 16)));
      em_free(&e, small);
    }
    /* backward, reverse layer order */
    for (int64_t l = L - 1; l >= 0; --l) {
      int32_t t0 = em_alloc(&e, jitter(&r, asize[6]));
      for (int p = 0; p < NPARAM; ++p) {
        grads[l * NPARAM + p] = em_alloc(&e, psize[p]);
        if (p == 3) {
          int32_t t1 = em_alloc(&e, jitter(&r, asize[0]));
          em_free(&e, t1);
        }
      }
      em_free(&e, t0);
      for (int a = NACT - 1; a >= 0; --a) em_free(&e, acts[l * NACT + a]);
      int32_t t2 = em_alloc(&e, jitter(&r, asize[0]));
      em_free(&e, t2);
    }
    have_grads = 1;
    /* optimizer: state allocated once (first iteration), permanent */
    if (it == 0)
      for (int64_t l = 0; l < L; ++l)
        for (int p = 0; p < NPARAM; ++p) {
          em_alloc(&e, psize[p]);
          em_alloc(&e, psize[p]);
        }
    em_free(&e, batch);
  }
  free(acts);
  free(grads);
  return e.n;
}

typedef struct {
  int32_t first, n;
  const int64_t* offs;
  pm_req_t* out;
  int64_t* counts;
  volatile int32_t* next;
} SynthJob;

static void* synth_worker(void* arg) {
  SynthJob* j = (SynthJob*)arg;
  for (;;) {
    int32_t t = __atomic_fetch_add(j->next, 1, __ATOMIC_RELAXED);
    if (t >= j->n) break;
    if (j->out)
      pm_synth_trace(j->first + t, j->out + j->offs[t]);
    else
      j->counts[t] = pm_synth_trace(j->first + t, NULL);
  }
  return NULL;
}

static void run_jobs(SynthJob* job, int n_threads) {
  if (n_threads <= 1) {
    synth_worker(job);
    return;
  }
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)n_threads);
  for (int i = 0; i < n_threads; ++i) pthread_create(&th[i], NULL, synth_worker, job);
  for (int i = 0; i < n_threads; ++i) pthread_join(th[i], NULL);
  free(th);
}

/* counts[t] = requests of trace first+t */
void pm_synth_counts(int32_t first, int32_t n, int64_t* counts, int n_threads) {
  volatile int32_t next = 0;
  SynthJob job = {first, n, NULL, NULL, counts, &next};
  run_jobs(&job, n_threads);
}

/* fill out[offs[t] .. offs[t+1]) with trace first+t */
void pm_synth_fill(int32_t first, int32_t n, const int64_t* offs, pm_req_t* out,
                   int n_threads) {
  volatile int32_t next = 0;
  SynthJob job = {first, n, offs, out, NULL, &next};
  run_jobs(&job, n_threads);
}
