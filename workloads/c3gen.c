/*
 * C3 workload generator: 10^4 synthetic Llama-style
 * request-level training traces, trace i seeded
 * numpy.random.Generator(PCG64(1_000_003 + i)).
 *
 * The executable spec is oracle/c3gen.py (numpy); this file reproduces it bit
 * for bit in C so the sweep (~1e9 requests) generates in seconds on host
 * threads.  It restates the numpy pieces the spec draws through:
 *   - SeedSequence(seed).generate_state(4, uint64)  (entropy pool of 4 uint32
 *     words, hashmix / mix, INIT_A/MULT_A/INIT_B/MULT_B constants);
 *   - PCG64: 128-bit LCG, XSL-RR 64-bit output, state advanced before output,
 *     srandom(initstate, initseq) seeding;
 *   - next_uint32: low half of a 64-bit draw first, high half buffered;
 *   - Generator.random(): (next64 >> 11) * 2^-53;
 *   - Generator.integers(lo, hi) for ranges below 2^32: Lemire's bounded
 *     rejection on next_uint32 draws (rng = hi - lo - 1; rng == 0 draws nothing).
 * tests/test_c3gen.py pins the output to oracle/c3gen.py trace for trace.
 *
 * Requests are the packed 16 B records of include/peakmem_b200.h, handles
 * dense in allocation order.  Compiled into the engine's synth library
 * (paper_2504_03887_b200/lib/libpeakmem_synth.so) and, for the reference
 * bench arm, into oracle/lib/liboracle_replay.so.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "../include/peakmem_b200.h"

typedef unsigned __int128 u128;

/* ---- numpy SeedSequence (numpy/random/bit_generator.pyx) ---------------- */
#define SS_INIT_A 0x43b0d7e5u
#define SS_MULT_A 0x931e8875u
#define SS_INIT_B 0x8b51f9ddu
#define SS_MULT_B 0x58f38dedu
#define SS_MIX_L 0xca01f9ddu
#define SS_MIX_R 0x4973f715u
#define SS_POOL 4

static uint32_t ss_hashmix(uint32_t v, uint32_t* hc) {
  v ^= *hc;
  *hc *= SS_MULT_A;
  v *= *hc;
  v ^= v >> 16;
  return v;
}

static uint32_t ss_mix(uint32_t x, uint32_t y) {
  uint32_t r = SS_MIX_L * x - SS_MIX_R * y;
  r ^= r >> 16;
  return r;
}

/* state words of SeedSequence(seed).generate_state(4, np.uint64) */
static void seed_sequence_u64x4(uint64_t seed, uint64_t out[4]) {
  uint32_t ent[2];
  int n_ent = 0;
  /* _coerce_to_uint32_array: little-endian 32-bit words, at least one */
  ent[n_ent++] = (uint32_t)seed;
  if (seed >> 32) ent[n_ent++] = (uint32_t)(seed >> 32);
  uint32_t pool[SS_POOL];
  uint32_t hc = SS_INIT_A;
  for (int i = 0; i < SS_POOL; ++i) pool[i] = ss_hashmix(i < n_ent ? ent[i] : 0u, &hc);
  for (int s = 0; s < SS_POOL; ++s)
    for (int d = 0; d < SS_POOL; ++d)
      if (s != d) pool[d] = ss_mix(pool[d], ss_hashmix(pool[s], &hc));
  uint32_t w[8];
  uint32_t hb = SS_INIT_B;
  for (int i = 0; i < 8; ++i) {
    uint32_t v = pool[i % SS_POOL];
    v ^= hb;
    hb *= SS_MULT_B;
    v *= hb;
    v ^= v >> 16;
    w[i] = v;
  }
  for (int i = 0; i < 4; ++i) out[i] = (uint64_t)w[2 * i] | ((uint64_t)w[2 * i + 1] << 32);
}

/* ---- PCG64 (numpy/random/src/pcg64) -------------------------------------- */
typedef struct {
  u128 state, inc;
  int has32;
  uint32_t buf32;
} Pcg64;

static const u128 PCG_MULT =
    ((u128)0x2360ED051FC65DA4ull << 64) | (u128)0x4385DF649FCCF645ull;

static void pcg_step(Pcg64* g) { g->state = g->state * PCG_MULT + g->inc; }

static void pcg_seed(Pcg64* g, uint64_t seed) {
  uint64_t v[4];
  seed_sequence_u64x4(seed, v);
  u128 initstate = ((u128)v[0] << 64) | v[1];
  u128 initseq = ((u128)v[2] << 64) | v[3];
  g->state = 0;
  g->inc = (initseq << 1) | 1u;
  pcg_step(g);
  g->state += initstate;
  pcg_step(g);
  g->has32 = 0;
  g->buf32 = 0;
}

static uint64_t pcg_next64(Pcg64* g) {
  pcg_step(g);
  uint64_t hi = (uint64_t)(g->state >> 64), lo = (uint64_t)g->state;
  uint64_t x = hi ^ lo;
  unsigned rot = (unsigned)(hi >> 58);
  return (x >> rot) | (x << ((64 - rot) & 63));
}

static uint32_t pcg_next32(Pcg64* g) {
  if (g->has32) {
    g->has32 = 0;
    return g->buf32;
  }
  uint64_t n = pcg_next64(g);
  g->has32 = 1;
  g->buf32 = (uint32_t)(n >> 32);
  return (uint32_t)n;
}

/* Generator.random() */
static double np_random(Pcg64* g) { return (double)(pcg_next64(g) >> 11) * (1.0 / 9007199254740992.0); }

/* Generator.integers(lo, hi) (hi exclusive, hi - lo <= 2^32) */
static int64_t np_integers(Pcg64* g, int64_t lo, int64_t hi) {
  uint32_t rng = (uint32_t)(hi - lo - 1);
  if (rng == 0) return lo;
  if (rng == 0xFFFFFFFFu) return lo + (int64_t)pcg_next32(g);
  uint32_t excl = rng + 1u;
  uint64_t m = (uint64_t)pcg_next32(g) * excl;
  uint32_t left = (uint32_t)m;
  if (left < excl) {
    uint32_t thresh = (UINT32_MAX - rng) % excl;
    while (left < thresh) {
      m = (uint64_t)pcg_next32(g) * excl;
      left = (uint32_t)m;
    }
  }
  return lo + (int64_t)(m >> 32);
}

/* ---- the trace (oracle/c3gen.py::trace) ---------------------------------- */
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

static int64_t jitter(Pcg64* g, int64_t size) {
  if (np_random(g) < 0.1) {
    int64_t j = (int64_t)((double)size * (0.5 + np_random(g)));
    return j > 0 ? j : 1;
  }
  return size;
}

#define NPARAM 9
#define NACT 10

/* Generate trace `index`; returns its request count. */
int64_t pm_synth_trace(int32_t index, pm_req_t* out) {
  Pcg64 g;
  pcg_seed(&g, 1000003ull + (uint64_t)index);
  static const int64_t layers_c[] = {4, 8, 16, 32};
  static const int64_t hidden_c[] = {1024, 2048, 3072, 4096};
  static const int64_t seq_c[] = {256, 512, 1024, 2048};
  const int64_t L = layers_c[np_integers(&g, 0, 4)];
  const int64_t h = hidden_c[np_integers(&g, 0, 4)];
  const int64_t ffn = 256 * ((8 * h + 767) / 768);
  const int64_t heads = h / 128;
  const int64_t b = np_integers(&g, 1, 17);
  const int64_t s = seq_c[np_integers(&g, 0, 4)];
  const int64_t target = np_integers(&g, 90000, 110001);
  const int64_t E = 2; /* bf16 */

  const int64_t psize[NPARAM] = {h * h * E,   h * h * E,   h * h * E, h * h * E, h * ffn * E,
                                 h * ffn * E, h * ffn * E, h * E,     h * E};
  const int64_t asize[NACT] = {b * s * h * E,   b * s * h * E,   b * s * h * E,  b * s * h * E,
                               b * s * h * E,   b * s * h * E,   b * s * ffn * E, b * s * ffn * E,
                               b * s * ffn * E, b * heads * s * s * E};
  Emit e = {out, 0, 0};
  int32_t* acts = (int32_t*)malloc(sizeof(int32_t) * (size_t)(L * NACT));
  int32_t* grads = (int32_t*)malloc(sizeof(int32_t) * (size_t)(L * NPARAM));
  int have_grads = 0;

  for (int64_t l = 0; l < L; ++l) /* model load, reversed */
    for (int p = NPARAM - 1; p >= 0; --p) em_alloc(&e, psize[p]);

  for (int64_t it = 0; e.n < target; ++it) {
    if (have_grads) /* zero_grad */
      for (int64_t i = 0; i < L * NPARAM; ++i) em_free(&e, grads[i]);
    int32_t batch = em_alloc(&e, b * s * 8);
    for (int64_t l = 0; l < L; ++l) { /* forward */
      for (int a = 0; a < NACT; ++a) {
        acts[l * NACT + a] = em_alloc(&e, jitter(&g, asize[a]));
        if (a % 3 == 2) {
          int32_t t = em_alloc(&e, jitter(&g, a < 6 ? asize[0] : asize[6]));
          em_free(&e, t);
        }
      }
      int64_t k = np_integers(&g, 0, 16);
      int32_t small = em_alloc(&e, jitter(&g, 4096 + 512 * k));
      em_free(&e, small);
    }
    for (int64_t l = L - 1; l >= 0; --l) { /* backward */
      int32_t t0 = em_alloc(&e, jitter(&g, asize[6]));
      for (int p = 0; p < NPARAM; ++p) {
        grads[l * NPARAM + p] = em_alloc(&e, psize[p]);
        if (p == 3) {
          int32_t t1 = em_alloc(&e, jitter(&g, asize[0]));
          em_free(&e, t1);
        }
      }
      em_free(&e, t0);
      for (int a = NACT - 1; a >= 0; --a) em_free(&e, acts[l * NACT + a]);
      int32_t t2 = em_alloc(&e, jitter(&g, asize[0]));
      em_free(&e, t2);
    }
    have_grads = 1;
    if (it == 0) /* optimizer state, permanent */
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

/* raw PCG64 draws of a seed, for the generator's own unit test */
void pm_synth_pcg64_raw(uint64_t seed, int32_t n, uint64_t* out) {
  Pcg64 g;
  pcg_seed(&g, seed);
  for (int32_t i = 0; i < n; ++i) out[i] = pcg_next64(&g);
}

typedef struct {
  const int32_t* ids; /* trace ids, or NULL: first + t */
  int32_t first, n;
  const int64_t* offs;
  pm_req_t* out;
  int64_t* counts;
  int32_t* next;
} SynthJob;

static void* synth_worker(void* arg) {
  SynthJob* j = (SynthJob*)arg;
  for (;;) {
    int32_t t = __atomic_fetch_add(j->next, 1, __ATOMIC_RELAXED);
    if (t >= j->n) break;
    int32_t id = j->ids ? j->ids[t] : j->first + t;
    if (j->out)
      pm_synth_trace(id, j->out + j->offs[t]);
    else
      j->counts[t] = pm_synth_trace(id, NULL);
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
  int32_t next = 0;
  SynthJob job = {NULL, first, n, NULL, NULL, counts, &next};
  run_jobs(&job, n_threads);
}

/* fill out[offs[t] .. offs[t+1]) with trace first+t */
void pm_synth_fill(int32_t first, int32_t n, const int64_t* offs, pm_req_t* out,
                   int n_threads) {
  int32_t next = 0;
  SynthJob job = {NULL, first, n, offs, out, NULL, &next};
  run_jobs(&job, n_threads);
}

/* the same for an arbitrary list of trace ids (a shard or a sample) */
void pm_synth_counts_ids(const int32_t* ids, int32_t n, int64_t* counts, int n_threads) {
  int32_t next = 0;
  SynthJob job = {ids, 0, n, NULL, NULL, counts, &next};
  run_jobs(&job, n_threads);
}

void pm_synth_fill_ids(const int32_t* ids, int32_t n, const int64_t* offs, pm_req_t* out,
                       int n_threads) {
  int32_t next = 0;
  SynthJob job = {ids, 0, n, offs, out, NULL, &next};
  run_jobs(&job, n_threads);
}
