/* TEST INFRASTRUCTURE ONLY — see mics_oracle.h.  Plain-C restatement of the
 * reference hot path; the checker, never the thing measured or shipped. */
#include "mics_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

enum { ORA_OK = 0, ORA_OUT_OF_RANGE = 1, ORA_NON_DIVISIBLE = 2, ORA_INFEASIBLE = 3,
       ORA_SIZE_MISMATCH = 4, ORA_TYPE_MISMATCH = 5, ORA_SHAPE_ERROR = 6 };

/* ------------------------------------------------------------------------
 * std::mt19937 (the generator every reference test seeds, e.g.
 * test_collectives.cpp:13-21) and the GCC 13 libstdc++ distributions.
 * ---------------------------------------------------------------------- */
typedef struct { uint32_t mt[624]; int idx; } mt_t;

static void mt_seed(mt_t* s, uint32_t seed) {
  s->mt[0] = seed;
  for (int i = 1; i < 624; ++i) s->mt[i] = 1812433253u * (s->mt[i - 1] ^ (s->mt[i - 1] >> 30)) + (uint32_t)i;
  s->idx = 624;
}

static uint32_t mt_next(mt_t* s) {
  if (s->idx >= 624) {
    for (int i = 0; i < 624; ++i) {
      uint32_t y = (s->mt[i] & 0x80000000u) | (s->mt[(i + 1) % 624] & 0x7fffffffu);
      s->mt[i] = s->mt[(i + 397) % 624] ^ (y >> 1) ^ ((y & 1u) ? 0x9908b0dfu : 0u);
    }
    s->idx = 0;
  }
  uint32_t y = s->mt[s->idx++];
  y ^= y >> 11;
  y ^= (y << 7) & 0x9d2c5680u;
  y ^= (y << 15) & 0xefc60000u;
  y ^= y >> 18;
  return y;
}

void ora_mt_random_shards(int count, size_t chunk, uint32_t seed, uint8_t* out) {
  mt_t s;
  mt_seed(&s, seed);
  for (size_t i = 0; i < (size_t)count * chunk; ++i) out[i] = (uint8_t)(mt_next(&s) & 0xffu);
}

/* uniform_int_distribution<int64_t>::operator() with a 32-bit URNG:
 * downscaling through Lemire's nearly-divisionless method (_S_nd<uint64_t>). */
static int64_t mt_uniform_i64(mt_t* s, int64_t lo, int64_t hi) {
  const uint64_t urange = (uint64_t)hi - (uint64_t)lo;
  if (urange >= 0xffffffffull) abort(); /* upscaling path: never used by the reference tests */
  const uint32_t range = (uint32_t)(urange + 1);
  uint64_t product = (uint64_t)mt_next(s) * range;
  uint32_t low = (uint32_t)product;
  if (low < range) {
    const uint32_t threshold = (uint32_t)(-range) % range;
    while (low < threshold) {
      product = (uint64_t)mt_next(s) * range;
      low = (uint32_t)product;
    }
  }
  return (int64_t)((uint64_t)lo + (product >> 32));
}

/* uniform_real_distribution<float>: generate_canonical<float,24> (one 32-bit
 * draw, divided by 2^32, clamped below 1) then x*(b-a)+a in float. */
static float mt_uniform_f32(mt_t* s, float lo, float hi) {
  float sum = 0.0f + (float)mt_next(s) * 1.0f;
  float ret = sum / 4294967296.0f;
  if (ret >= 1.0f) ret = nextafterf(1.0f, 0.0f);
  return ret * (hi - lo) + lo;
}

void ora_mt_random_i64(size_t count, int64_t lo, int64_t hi, uint32_t seed, int64_t* out) {
  mt_t s;
  mt_seed(&s, seed);
  for (size_t i = 0; i < count; ++i) out[i] = mt_uniform_i64(&s, lo, hi);
}

void ora_mt_random_f32(size_t count, float lo, float hi, uint32_t seed, float* out) {
  mt_t s;
  mt_seed(&s, seed);
  for (size_t i = 0; i < count; ++i) out[i] = mt_uniform_f32(&s, lo, hi);
}

uint64_t ora_splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static uint64_t gen_key(uint64_t seed, int rank, int step, int layer, uint64_t idx) {
  return seed ^ ((uint64_t)rank << 40) ^ ((uint64_t)step << 32) ^ ((uint64_t)layer << 24) ^ idx;
}

void ora_gen_f32(uint64_t seed, int rank, int step, int layer, uint64_t start, size_t count, float* out) {
  for (size_t i = 0; i < count; ++i) {
    uint64_t x = ora_splitmix64(gen_key(seed, rank, step, layer, start + i));
    out[i] = (float)((int32_t)(x >> 40) - (1 << 23)) * (1.0f / 8388608.0f);
  }
}

void ora_gen_bf16(uint64_t seed, int rank, int step, int layer, uint64_t start, size_t count, uint16_t* out) {
  for (size_t i = 0; i < count; ++i) {
    uint64_t x = ora_splitmix64(gen_key(seed, rank, step, layer, start + i));
    float f = (float)((int32_t)(x >> 56) - 128) * (1.0f / 128.0f);
    uint32_t b;
    memcpy(&b, &f, 4);
    out[i] = (uint16_t)(b >> 16); /* exact: 8 significant bits */
  }
}

/* ------------------------------------------------------------------------
 * topology (topology.cpp:21-84)
 * ---------------------------------------------------------------------- */
int ora_build_group_layout(int n, int p, int* part, int* repl) {
  if (p < 1 || p > n) return ORA_OUT_OF_RANGE; /* topology.cpp:22-24 */
  if (n % p != 0) return ORA_NON_DIVISIBLE;    /* topology.cpp:25-27 */
  int i = 0;
  for (int g = 0; g < n / p; ++g)
    for (int j = 0; j < p; ++j) part[i++] = g * p + j; /* contiguous ranges, :33-36 */
  i = 0;
  for (int j = 0; j < p; ++j)
    for (int r = j; r < n; r += p) repl[i++] = r; /* stride-p sets, :38-41 */
  return ORA_OK;
}

int ora_partition_shape_ok(int p, int k) { /* topology.cpp:45-49 */
  if (p < 1 || k < 1) return 0;
  if (p <= k) return k % p == 0;
  return p % k == 0;
}

int ora_min_feasible_partition(uint64_t state_bytes, int num_nodes, int k, uint64_t device_memory,
                               int node_granular, double headroom, int* out) {
  if (state_bytes == 0 || num_nodes < 1 || k < 1) return ORA_OUT_OF_RANGE; /* :61-63 + validate */
  const int n = num_nodes * k;
  const double budget = (double)device_memory * headroom;
  for (int p = 1; p <= n; ++p) { /* :68-80: smallest admissible p whose share fits */
    if (n % p) continue;
    if (node_granular) {
      if (p % k) continue;
    } else if (!ora_partition_shape_ok(p, k)) {
      continue;
    }
    if ((double)state_bytes / (double)p <= budget) {
      *out = p;
      return ORA_OK;
    }
  }
  return ORA_INFEASIBLE;
}

/* ------------------------------------------------------------------------
 * collectives (collectives.cpp:81-291)
 * ---------------------------------------------------------------------- */
static size_t dsize(int dtype) { return dtype == 1 ? 4 : 8; }

/* acc[e] = acc[e] + src[e] in T (collectives.cpp:81-99) */
static void accumulate(uint8_t* acc, const uint8_t* src, size_t bytes, int dtype) {
  if (dtype == 0) {
    for (size_t e = 0; e < bytes / 8; ++e) {
      int64_t a, b;
      memcpy(&a, acc + 8 * e, 8);
      memcpy(&b, src + 8 * e, 8);
      a = (int64_t)((uint64_t)a + (uint64_t)b); /* two's-complement wrap */
      memcpy(acc + 8 * e, &a, 8);
    }
  } else if (dtype == 1) {
    for (size_t e = 0; e < bytes / 4; ++e) {
      float a, b;
      memcpy(&a, acc + 4 * e, 4);
      memcpy(&b, src + 4 * e, 4);
      a = a + b;
      memcpy(acc + 4 * e, &a, 4);
    }
  } else {
    for (size_t e = 0; e < bytes / 8; ++e) {
      double a, b;
      memcpy(&a, acc + 8 * e, 8);
      memcpy(&b, src + 8 * e, 8);
      a = a + b;
      memcpy(acc + 8 * e, &a, 8);
    }
  }
}

/* out[j] = C_0 || ... || C_{p-1} for every position j (collectives.cpp:103-134) */
int ora_all_gather(int p, const uint8_t* shards, size_t chunk, uint8_t* out) {
  for (int j = 0; j < p; ++j) memcpy(out + (size_t)j * p * chunk, shards, (size_t)p * chunk);
  return ORA_OK;
}

/* position j gets fold_{i=0..p-1} buffers[i][j-th chunk], ascending position,
 * starting from position 0's value (collectives.cpp:136-183) */
int ora_reduce_scatter(int p, const uint8_t* bufs, size_t bytes, int dtype, uint8_t* out) {
  if (p < 1) return ORA_OK;
  if (bytes % ((size_t)p * dsize(dtype))) return ORA_TYPE_MISMATCH; /* :148-153 */
  const size_t chunk = bytes / p;
  for (int j = 0; j < p; ++j) {
    uint8_t* o = out + (size_t)j * chunk;
    memcpy(o, bufs + (size_t)j * chunk, chunk); /* contribution(0) = buffers[0], chunk j */
    for (int i = 1; i < p; ++i) accumulate(o, bufs + (size_t)i * bytes + (size_t)j * chunk, chunk, dtype);
  }
  return ORA_OK;
}

/* reduce_scatter then all_gather (collectives.cpp:185-190) */
int ora_all_reduce(int p, const uint8_t* bufs, size_t bytes, int dtype, uint8_t* out) {
  if (p < 1) return ORA_OK;
  uint8_t* rs = (uint8_t*)malloc(bytes ? bytes : 1);
  int st = ora_reduce_scatter(p, bufs, bytes, dtype, rs);
  if (st == ORA_OK) ora_all_gather(p, rs, bytes / p, out);
  free(rs);
  return st;
}

/* Three-stage hierarchical all-gather over every partition group
 * (collectives.cpp:192-291).  shards: n x chunk by global rank; out: n x p*chunk. */
int ora_hier_all_gather(int n, int p, int k, const uint8_t* shards, size_t chunk, int corrupt, uint8_t* out) {
  if (p < 1 || p > n || n % p) return p < 1 || p > n ? ORA_OUT_OF_RANGE : ORA_NON_DIVISIBLE;
  if (n % k) return ORA_SHAPE_ERROR;
  if (!ora_partition_shape_ok(p, k)) return ORA_SHAPE_ERROR; /* :208-210 */
  const size_t row = (size_t)p * chunk;
  for (int g = 0; g < n / p; ++g) {
    const int base = g * p;
    if (p <= k) { /* :218-225 plain all-gather */
      for (int i = 0; i < p; ++i) memcpy(out + (size_t)(base + i) * row, shards + (size_t)base * chunk, row);
      continue;
    }
    const int q = p / k;
    /* stage 1 (:232-241): member (m, j) ends with [C_j, C_{k+j}, ..., C_{(q-1)k+j}] */
    uint8_t* stage1 = (uint8_t*)malloc((size_t)k * q * chunk + 1); /* identical on every member of channel j */
    for (int j = 0; j < k; ++j)
      for (int m = 0; m < q; ++m)
        memcpy(stage1 + ((size_t)j * q + m) * chunk, shards + (size_t)(base + m * k + j) * chunk, chunk);
    for (int m = 0; m < q; ++m) {
      for (int j = 0; j < k; ++j) {
        uint8_t* o = out + (size_t)(base + m * k + j) * row;
        if (corrupt) { /* :243-256 gather the raw stage-1 buffers per node */
          for (int jj = 0; jj < k; ++jj) memcpy(o + (size_t)jj * q * chunk, stage1 + (size_t)jj * q * chunk, (size_t)q * chunk);
        } else { /* :259-288 stage 2 picks chunk t of every local rank's stage-1
                    buffer, stage 3 gathers batch t at offset t*k*chunk */
          for (int t = 0; t < q; ++t)
            for (int jj = 0; jj < k; ++jj)
              memcpy(o + ((size_t)t * k + jj) * chunk, stage1 + ((size_t)jj * q + t) * chunk, chunk);
        }
      }
    }
    free(stage1);
  }
  return ORA_OK;
}

/* record_traffic(from, to, chunk) for every ordered pair (collectives.cpp:116-123, :157-165) */
static void traffic_pairs(const int* ranks, int p, uint64_t bytes, int n, uint64_t* mat) {
  for (int i = 0; i < p; ++i)
    for (int j = 0; j < p; ++j)
      if (i != j) mat[(size_t)ranks[i] * n + ranks[j]] += bytes;
}

void ora_traffic_all_gather(const int* ranks, int p, size_t chunk, int n, uint64_t* mat) {
  traffic_pairs(ranks, p, chunk, n, mat);
}
void ora_traffic_reduce_scatter(const int* ranks, int p, size_t bytes, int n, uint64_t* mat) {
  if (p > 0) traffic_pairs(ranks, p, bytes / p, n, mat);
}
void ora_traffic_all_reduce(const int* ranks, int p, size_t bytes, int n, uint64_t* mat) {
  if (p > 0) {
    traffic_pairs(ranks, p, bytes / p, n, mat);
    traffic_pairs(ranks, p, bytes / p, n, mat);
  }
}

int ora_traffic_hier_all_gather(int n, int p, int k, size_t chunk, int corrupt, uint64_t* mat) {
  if (p < 1 || p > n || n % p || !ora_partition_shape_ok(p, k)) return ORA_SHAPE_ERROR;
  int* rk = (int*)malloc(sizeof(int) * (size_t)(p + k + 1));
  for (int g = 0; g < n / p; ++g) {
    const int base = g * p;
    if (p <= k) {
      for (int i = 0; i < p; ++i) rk[i] = base + i;
      traffic_pairs(rk, p, chunk, n, mat);
      continue;
    }
    const int q = p / k;
    for (int j = 0; j < k; ++j) { /* stage 1 channels */
      for (int m = 0; m < q; ++m) rk[m] = base + m * k + j;
      traffic_pairs(rk, q, chunk, n, mat);
    }
    for (int m = 0; m < q; ++m) { /* stage 3 (or the corrupt node gather of q*chunk) */
      for (int j = 0; j < k; ++j) rk[j] = base + m * k + j;
      if (corrupt)
        traffic_pairs(rk, k, (uint64_t)q * chunk, n, mat);
      else
        for (int t = 0; t < q; ++t) traffic_pairs(rk, k, chunk, n, mat);
    }
  }
  free(rk);
  return ORA_OK;
}

/* ------------------------------------------------------------------------
 * sync schedule (sync_schedule.hpp:45-256)
 * ---------------------------------------------------------------------- */
typedef struct {
  int64_t* ev;
  int cap;
  int n;
} evlog_t;

static void log_event(evlog_t* L, int step, int phase, int group, uint64_t bytes) {
  if (L->ev && L->n < L->cap) {
    L->ev[4 * L->n + 0] = step;
    L->ev[4 * L->n + 1] = phase;
    L->ev[4 * L->n + 2] = group;
    L->ev[4 * L->n + 3] = (int64_t)bytes;
  }
  L->n++;
}

static int check_layout(int n, int p) {
  if (p < 1 || p > n) return ORA_OUT_OF_RANGE;
  if (n % p) return ORA_NON_DIVISIBLE;
  return ORA_OK;
}

/* element (t, r, e) of the s x n x len gradient set, zero past len (padded_grad :105-111) */
static const uint8_t* grad_at(const uint8_t* g, size_t sz, int n, size_t len, int t, int r, size_t e) {
  static const uint8_t zero[8] = {0};
  if (e >= len) return zero;
  return g + (((size_t)t * n + r) * len + e) * sz;
}

int ora_two_hop(int dtype, int n, int p, int s, size_t len, const void* grads_v, void* out_v,
                int64_t* ev, int cap, int* nev, uint64_t* traffic) {
  int st = check_layout(n, p);
  if (st) return st;
  if (s < 1) return ORA_OUT_OF_RANGE; /* make_sync_states :61 */
  const uint8_t* grads = (const uint8_t*)grads_v;
  uint8_t* shard = (uint8_t*)out_v;
  const size_t sz = dsize(dtype);
  const size_t chunk = (len + p - 1) / p; /* owned_chunk_elems :53-56 */
  evlog_t L = {ev, cap, 0};
  memset(shard, 0, (size_t)n * chunk * sz); /* T{} */
  uint8_t* vals = (uint8_t*)malloc(chunk * sz + 8);
  int* rk = (int*)malloc(sizeof(int) * (size_t)n);
  /* micro-steps (:118-147): reduce-scatter inside each partition group, then shard += */
  for (int t = 0; t < s; ++t) {
    for (int g = 0; g < n / p; ++g) {
      for (int j = 0; j < p; ++j) {
        for (size_t e = 0; e < chunk; ++e) {
          const size_t x = (size_t)j * chunk + e;
          memcpy(vals + e * sz, grad_at(grads, sz, n, len, t, g * p + 0, x), sz);
          for (int i = 1; i < p; ++i) accumulate(vals + e * sz, grad_at(grads, sz, n, len, t, g * p + i, x), sz, dtype);
        }
        accumulate(shard + (size_t)(g * p + j) * chunk * sz, vals, chunk * sz, dtype);
      }
      if (traffic) {
        for (int i = 0; i < p; ++i) rk[i] = g * p + i;
        ora_traffic_reduce_scatter(rk, p, (size_t)p * chunk * sz, n, traffic);
      }
      log_event(&L, t, 0, g, (uint64_t)(p - 1) * chunk * sz);
    }
  }
  /* boundary (:153-185): all-reduce inside each replication group over the
   * shard padded to a multiple of r; the fold runs in ascending position. */
  const int r = n / p;
  const size_t padded = ((chunk + r - 1) / r) * r;
  for (int j = 0; j < p; ++j) {
    if (r > 1) {
      for (size_t e = 0; e < chunk; ++e) {
        memcpy(vals + e * sz, shard + ((size_t)j * chunk + e) * sz, sz);
        for (int i = 1; i < r; ++i) accumulate(vals + e * sz, shard + ((size_t)(j + i * p) * chunk + e) * sz, sz, dtype);
      }
      for (int i = 0; i < r; ++i) memcpy(shard + (size_t)(j + i * p) * chunk * sz, vals, chunk * sz);
      if (traffic) {
        for (int i = 0; i < r; ++i) rk[i] = j + i * p;
        ora_traffic_all_reduce(rk, r, padded * sz, n, traffic);
      }
    }
    log_event(&L, s, 1, j, (uint64_t)2 * (r - 1) * (padded / r) * sz);
  }
  free(vals);
  free(rk);
  if (nev) *nev = L.n;
  return ORA_OK;
}

int ora_alternative(int dtype, int n, int p, int s, size_t len, const void* grads_v, void* out_v,
                    int64_t* ev, int cap, int* nev, uint64_t* traffic) {
  int st = check_layout(n, p);
  if (st) return st;
  if (s < 1) return ORA_OUT_OF_RANGE;
  const uint8_t* grads = (const uint8_t*)grads_v;
  uint8_t* shard = (uint8_t*)out_v;
  const size_t sz = dsize(dtype);
  const size_t chunk = (len + p - 1) / p;
  const size_t elems = chunk * p;
  const size_t padded = ((elems + n - 1) / n) * n; /* :200-201 */
  evlog_t L = {ev, cap, 0};
  memset(shard, 0, (size_t)n * chunk * sz);
  uint8_t* red = (uint8_t*)malloc(elems * sz + 8);
  int* rk = (int*)malloc(sizeof(int) * (size_t)n);
  for (int i = 0; i < n; ++i) rk[i] = i;
  for (int t = 0; t < s; ++t) { /* :189-224 all-reduce over all n, keep owned chunk */
    for (size_t x = 0; x < elems; ++x) {
      memcpy(red + x * sz, grad_at(grads, sz, n, len, t, 0, x), sz);
      for (int i = 1; i < n; ++i) accumulate(red + x * sz, grad_at(grads, sz, n, len, t, i, x), sz, dtype);
    }
    for (int rr = 0; rr < n; ++rr)
      accumulate(shard + (size_t)rr * chunk * sz, red + (size_t)(rr % p) * chunk * sz, chunk * sz, dtype);
    if (traffic) ora_traffic_all_reduce(rk, n, padded * sz, n, traffic);
    log_event(&L, t, 2, 0, (uint64_t)2 * (n - 1) * (padded / n) * sz);
  }
  free(red);
  free(rk);
  if (nev) *nev = L.n;
  return ORA_OK;
}

/* step-major scalar sum sliced by ownership (:236-256) */
int ora_global_sync(int dtype, int n, int p, int s, size_t len, const void* grads_v, void* out_v) {
  int st = check_layout(n, p);
  if (st) return st;
  const uint8_t* grads = (const uint8_t*)grads_v;
  const size_t sz = dsize(dtype);
  const size_t chunk = (len + p - 1) / p;
  uint8_t* total = (uint8_t*)calloc(chunk * p + 1, sz);
  for (int t = 0; t < s; ++t)
    for (int r = 0; r < n; ++r)
      for (size_t e = 0; e < len; ++e) accumulate(total + e * sz, grad_at(grads, sz, n, len, t, r, e), sz, dtype);
  for (int r = 0; r < n; ++r) memcpy((uint8_t*)out_v + (size_t)r * chunk * sz, total + (size_t)(r % p) * chunk * sz, chunk * sz);
  free(total);
  return ORA_OK;
}

/* ------------------------------------------------------------------------
 * sharded Adam (no reference code; documented formula, see header)
 * ---------------------------------------------------------------------- */
void ora_adam_scalars(double lr, double b1, double b2, double eps, double wd, int step, double grad_scale,
                      ora_adam_scalars_t* o) {
  const double bc1 = 1.0 - pow(b1, (double)step);
  const double bc2 = 1.0 - pow(b2, (double)step);
  o->b1 = (float)b1;
  o->omb1 = (float)(1.0 - b1);
  o->b2 = (float)b2;
  o->omb2 = (float)(1.0 - b2);
  o->eps = (float)eps;
  o->wd = (float)wd;
  o->step_size = (float)(lr / bc1);
  o->bc2_sqrt = (float)sqrt(bc2);
  o->grad_scale = (float)grad_scale;
}

uint16_t ora_f32_to_bf16(float x) { /* round to nearest even; NaN kept quiet */
  uint32_t b;
  memcpy(&b, &x, 4);
  if ((b & 0x7fffffffu) > 0x7f800000u) return (uint16_t)((b >> 16) | 0x40u);
  b += 0x7fffu + ((b >> 16) & 1u);
  return (uint16_t)(b >> 16);
}

void ora_adam_f32(size_t count, float* param, float* m, float* v, const float* grad,
                  const ora_adam_scalars_t* sc, uint16_t* param_bf16) {
  for (size_t i = 0; i < count; ++i) {
    float g = grad[i] * sc->grad_scale;
    float p = param[i];
    if (sc->wd != 0.0f) g = g + sc->wd * p;
    float mi = sc->b1 * m[i] + sc->omb1 * g;
    float vi = sc->b2 * v[i] + sc->omb2 * (g * g);
    float denom = sqrtf(vi) / sc->bc2_sqrt + sc->eps;
    p = p - sc->step_size * (mi / denom);
    m[i] = mi;
    v[i] = vi;
    param[i] = p;
    if (param_bf16) param_bf16[i] = ora_f32_to_bf16(p);
  }
}

/* ------------------------------------------------------------------------
 * whole-shard expected step (see the header): test infrastructure for the
 * full-size bit-exact check of the step driver
 * ---------------------------------------------------------------------- */
typedef struct {
  uint64_t seed;
  int n, p, s, j;
  const ora_seg_t* segs;
  int nseg;
  uint64_t lo, hi;
  ora_adam_scalars_t sc;
  float *master, *m, *v;
  uint16_t* bf16;
} step1_job_t;

static float gen_one(uint64_t seed, int rank, int step, int layer, uint64_t idx) {
  const uint64_t x = ora_splitmix64(gen_key(seed, rank, step, layer, idx));
  return (float)((int32_t)(x >> 40) - (1 << 23)) * (1.0f / 8388608.0f);
}

static void* step1_worker(void* arg) {
  const step1_job_t* J = (const step1_job_t*)arg;
  const int r = J->n / J->p;
  int q = 0;
  while (q + 1 < J->nseg && J->segs[q + 1].so <= J->lo) ++q;
  for (uint64_t x = J->lo; x < J->hi; ++x) {
    while (q + 1 < J->nseg && J->segs[q + 1].so <= x) ++q;
    const ora_seg_t* S = &J->segs[q];
    const uint64_t pos = (uint64_t)J->j * S->c + (x - S->so), gi = S->go + pos;
    const int valid = pos < S->len;
    float red = 0.0f;
    for (int gg = 0; gg < r; ++gg) { /* replica gg: partition group gg */
      float acc = 0.0f;
      for (int t = 0; t < J->s; ++t) {
        float f = 0.0f;
        if (valid) {
          f = gen_one(J->seed, gg * J->p, t, 0, gi);
          for (int i = 1; i < J->p; ++i) f = f + gen_one(J->seed, gg * J->p + i, t, 0, gi);
        }
        acc = t ? acc + f : 0.0f + f;
      }
      red = gg ? red + acc : acc;
    }
    float pm = gen_one(J->seed ^ 0x5EEDull, J->j, 0, 255, x), mm = 0.0f, vv = 0.0f;
    uint16_t b;
    ora_adam_f32(1, &pm, &mm, &vv, &red, &J->sc, &b);
    J->master[x] = pm;
    J->m[x] = mm;
    J->v[x] = vv;
    J->bf16[x] = b;
  }
  return NULL;
}

int ora_step1_shard(uint64_t seed, int n, int p, int s, int j, const ora_seg_t* segs, int nseg, uint64_t shard_elems,
                    double lr, double b1, double b2, double eps, double wd, int threads, float* master, float* m,
                    float* v, uint16_t* bf16) {
  if (n <= 0 || p <= 0 || n % p || j < 0 || j >= p || nseg <= 0 || threads <= 0) return 1;
  if (threads > 256) threads = 256;
  pthread_t th[256];
  step1_job_t jobs[256];
  ora_adam_scalars_t sc;
  ora_adam_scalars(lr, b1, b2, eps, wd, 1, 1.0 / ((double)n * s), &sc);
  const uint64_t per = (shard_elems + threads - 1) / threads;
  int started = 0;
  for (int k = 0; k < threads; ++k) {
    step1_job_t* J = &jobs[k];
    J->seed = seed; J->n = n; J->p = p; J->s = s; J->j = j; J->segs = segs; J->nseg = nseg;
    J->lo = (uint64_t)k * per;
    J->hi = J->lo + per < shard_elems ? J->lo + per : shard_elems;
    J->sc = sc; J->master = master; J->m = m; J->v = v; J->bf16 = bf16;
    if (J->lo >= J->hi) break;
    if (pthread_create(&th[k], NULL, step1_worker, J)) return 2;
    ++started;
  }
  for (int k = 0; k < started; ++k) pthread_join(th[k], NULL);
  return 0;
}
