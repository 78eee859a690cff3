/*
 * relay_oracle.c -- CPU restatement of the reference relay-prefill hot path.
 *
 * TEST INFRASTRUCTURE ONLY (the checker, never the product path). Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load
 * build/liboracle.so.
 *
 * Plain C11 compiled with -ffp-contract=off, like the reference
 * (proj/src/CMakeLists.txt:16-18), so every float expression rounds exactly
 * as the reference's. Each function cites the reference file:line it
 * restates (paths relative to /root/reference/proj). The restatement is
 * pinned bit-for-bit against the reference itself (oracle/_ref, built from
 * the reference sources) by tests/test_oracle_pins.py and against the
 * committed golden vectors in tests/golden/ (made by
 * tests/golden/make_golden.py from oracle/_ref).
 *
 * Error behaviour: the same conditions the reference throws on return the
 * rk_status code of that exception type (include/relaykv_b200.h), with the
 * reference's message in orc_last_error().
 */
#define _POSIX_C_SOURCE 199309L
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#include "relaykv_b200.h"

static char g_err[512];
static int fail(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}
const char* orc_last_error(void) { return g_err; }

static double now_ms(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return ts.tv_sec * 1e3 + ts.tv_nsec * 1e-6;
}

/* ------------------------------------------------------------------------ */
/* weights: init_weights (src/model.cpp:81-114), SplitMix64 (model.cpp:49-62) */
/* ------------------------------------------------------------------------ */

typedef struct {
  float *attn_norm, *wq, *wk, *wv, *wo, *mlp_norm, *wgate, *wup, *wdown;
} orc_layer;

typedef struct orc_weights {
  rk_model_spec s;
  float* emb;
  orc_layer* layers;
  float* final_norm;
  float* head;
} orc_weights;

static uint64_t mix_next(uint64_t* state) {
  uint64_t z = (*state += 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
static float mix_symmetric(uint64_t* state) { /* model.cpp:57-60 */
  const float u = (float)(mix_next(state) >> 40) * 0x1p-24f;
  return 2.0f * u - 1.0f;
}
static float* uniform_tensor(uint64_t* rng, size_t n, float sd) { /* model.cpp:66-71 */
  float* t = (float*)malloc(n * sizeof(float));
  const float scale = sd * 1.7320508f;
  for (size_t i = 0; i < n; ++i) t[i] = mix_symmetric(rng) * scale;
  return t;
}
static float* ones_tensor(size_t n) {
  float* t = (float*)malloc(n * sizeof(float));
  for (size_t i = 0; i < n; ++i) t[i] = 1.0f;
  return t;
}

/* init_weights without spec.validate() (model.cpp:82). */
orc_weights* orc_weights_init(const rk_model_spec* spec, uint64_t seed) {
  orc_weights* w = (orc_weights*)calloc(1, sizeof *w);
  const rk_model_spec s = *spec;
  w->s = s;
  uint64_t rng = seed ^ 0x72656c6179ull;
  const size_t d = s.d_model, q = s.num_heads * s.d_head, kv = s.num_kv_heads * s.d_head;
  w->emb = uniform_tensor(&rng, s.vocab_size * d, 0.02f);
  const float d_in = 1.0f / sqrtf((float)d);
  const float ff_in = 1.0f / sqrtf((float)s.d_ff);
  const float q_in = 1.0f / sqrtf((float)q) / (2.0f * (float)s.num_layers);
  w->layers = (orc_layer*)calloc(s.num_layers, sizeof(orc_layer));
  for (size_t l = 0; l < s.num_layers; ++l) {
    orc_layer* L = &w->layers[l];
    L->attn_norm = ones_tensor(d);
    L->wq = uniform_tensor(&rng, d * q, d_in);
    L->wk = uniform_tensor(&rng, d * kv, d_in);
    L->wv = uniform_tensor(&rng, d * kv, d_in);
    L->wo = uniform_tensor(&rng, q * d, q_in);
    L->mlp_norm = ones_tensor(d);
    L->wgate = uniform_tensor(&rng, d * s.d_ff, d_in);
    L->wup = uniform_tensor(&rng, d * s.d_ff, d_in);
    L->wdown = uniform_tensor(&rng, s.d_ff * d, ff_in);
  }
  w->final_norm = ones_tensor(d);
  w->head = uniform_tensor(&rng, d * s.vocab_size, d_in);
  return w;
}

void orc_weights_destroy(orc_weights* w) {
  if (!w) return;
  for (size_t l = 0; l < w->s.num_layers; ++l) {
    orc_layer* L = &w->layers[l];
    free(L->attn_norm); free(L->wq); free(L->wk); free(L->wv); free(L->wo);
    free(L->mlp_norm); free(L->wgate); free(L->wup); free(L->wdown);
  }
  free(w->layers); free(w->emb); free(w->final_norm); free(w->head); free(w);
}

/* tensor_table order (src/weights_io.cpp:21-38). */
const float* orc_weights_tensor(orc_weights* w, uint64_t idx, uint64_t* numel) {
  const rk_model_spec s = w->s;
  const size_t d = s.d_model, q = s.num_heads * s.d_head, kv = s.num_kv_heads * s.d_head;
  if (idx == 0) { *numel = s.vocab_size * d; return w->emb; }
  idx -= 1;
  if (idx < 9 * s.num_layers) {
    orc_layer* L = &w->layers[idx / 9];
    switch (idx % 9) {
      case 0: *numel = d; return L->attn_norm;
      case 1: *numel = d * q; return L->wq;
      case 2: *numel = d * kv; return L->wk;
      case 3: *numel = d * kv; return L->wv;
      case 4: *numel = q * d; return L->wo;
      case 5: *numel = d; return L->mlp_norm;
      case 6: *numel = d * s.d_ff; return L->wgate;
      case 7: *numel = d * s.d_ff; return L->wup;
      default: *numel = s.d_ff * d; return L->wdown;
    }
  }
  idx -= 9 * s.num_layers;
  if (idx == 0) { *numel = d; return w->final_norm; }
  *numel = d * s.vocab_size;
  return w->head;
}

/* ------------------------------------------------------------------------ */
/* fp32 kernels (src/tensor.cpp)                                             */
/* ------------------------------------------------------------------------ */

static int g_nonfinite;

/* matmul (tensor.cpp:66-86): i-k-j, per element sequential k from 0.0f,
 * multiply then add (no FMA); ensure_finite (58-64) afterwards. */
static void matmul(const float* a, size_t m, size_t k, const float* b, size_t n, float* out) {
  memset(out, 0, m * n * sizeof(float));
  for (size_t i = 0; i < m; ++i) {
    const float* arow = a + i * k;
    float* orow = out + i * n;
    for (size_t kk = 0; kk < k; ++kk) {
      const float av = arow[kk];
      const float* brow = b + kk * n;
      for (size_t j = 0; j < n; ++j) orow[j] += av * brow[j];
    }
  }
  for (size_t i = 0; i < m * n; ++i)
    if (!isfinite(out[i])) g_nonfinite = 1;
}

/* softmax_inplace (tensor.cpp:88-98). */
static void softmax_inplace(float* row, size_t n) {
  if (n == 0) return;
  float mx = row[0];
  for (size_t i = 0; i < n; ++i) mx = (mx < row[i]) ? row[i] : mx;
  float sum = 0.0f;
  for (size_t i = 0; i < n; ++i) {
    row[i] = expf(row[i] - mx);
    sum += row[i];
  }
  for (size_t i = 0; i < n; ++i) row[i] /= sum;
}

/* rms_norm (tensor.cpp:109-119). */
static void rms_norm(const float* x, const float* gain, float eps, size_t n, float* out) {
  float ms = 0.0f;
  for (size_t i = 0; i < n; ++i) ms += x[i] * x[i];
  ms /= (float)n;
  const float inv = 1.0f / sqrtf(ms + eps);
  for (size_t i = 0; i < n; ++i) out[i] = x[i] * inv * gain[i];
}

/* rope_rotate (tensor.cpp:128-143): adjacent pairs, angle and products in double. */
static void rope_rotate(float* x, size_t n, int64_t position, float theta_base) {
  const double d = (double)n;
  for (size_t i = 0; i < n / 2; ++i) {
    const double freq = pow((double)theta_base, -2.0 * (double)i / d);
    const double angle = (double)position * freq;
    const double c = cos(angle), s = sin(angle);
    const double x0 = x[2 * i], x1 = x[2 * i + 1];
    x[2 * i] = (float)(c * x0 - s * x1);
    x[2 * i + 1] = (float)(s * x0 + c * x1);
  }
}
/* rope_rotate_heads (model.cpp:163-168). */
static void rope_rotate_heads(float* row, size_t heads, size_t dh, int64_t pos, float theta) {
  for (size_t h = 0; h < heads; ++h) rope_rotate(row + h * dh, dh, pos, theta);
}

/* ------------------------------------------------------------------------ */
/* KVContext (model.hpp:68-87, model.cpp:120-143) + SegmentMarks list         */
/* ------------------------------------------------------------------------ */

typedef struct {
  uint64_t base, len;
  uint8_t* origin; /* [L x len] layer-major */
} orc_marks;

typedef struct orc_ctx {
  size_t L, kv, size, cap;
  float** k;
  float** v;
  orc_marks* segs;
  size_t nsegs;
} orc_ctx;

orc_ctx* orc_ctx_create(orc_weights* w) {
  orc_ctx* c = (orc_ctx*)calloc(1, sizeof *c);
  c->L = w->s.num_layers;
  c->kv = w->s.num_kv_heads * w->s.d_head;
  c->k = (float**)calloc(c->L, sizeof(float*));
  c->v = (float**)calloc(c->L, sizeof(float*));
  return c;
}
void orc_ctx_destroy(orc_ctx* c) {
  if (!c) return;
  for (size_t l = 0; l < c->L; ++l) { free(c->k[l]); free(c->v[l]); }
  for (size_t i = 0; i < c->nsegs; ++i) free(c->segs[i].origin);
  free(c->k); free(c->v); free(c->segs); free(c);
}
static void ctx_resize(orc_ctx* c, size_t positions) { /* grows zero-filled */
  if (positions <= c->size) return;
  if (positions > c->cap) {
    size_t cap = c->cap ? c->cap : 64;
    while (cap < positions) cap *= 2;
    for (size_t l = 0; l < c->L; ++l) {
      c->k[l] = (float*)realloc(c->k[l], cap * c->kv * sizeof(float));
      c->v[l] = (float*)realloc(c->v[l], cap * c->kv * sizeof(float));
    }
    c->cap = cap;
  }
  for (size_t l = 0; l < c->L; ++l) {
    memset(c->k[l] + c->size * c->kv, 0, (positions - c->size) * c->kv * sizeof(float));
    memset(c->v[l] + c->size * c->kv, 0, (positions - c->size) * c->kv * sizeof(float));
  }
  c->size = positions;
}
static float* krow(orc_ctx* c, size_t l, size_t p) { return c->k[l] + p * c->kv; }
static float* vrow(orc_ctx* c, size_t l, size_t p) { return c->v[l] + p * c->kv; }

orc_ctx* orc_ctx_clone(orc_ctx* src) {
  orc_ctx* c = (orc_ctx*)calloc(1, sizeof *c);
  c->L = src->L; c->kv = src->kv;
  c->k = (float**)calloc(c->L, sizeof(float*));
  c->v = (float**)calloc(c->L, sizeof(float*));
  ctx_resize(c, src->size);
  for (size_t l = 0; l < c->L; ++l) {
    memcpy(c->k[l], src->k[l], src->size * c->kv * sizeof(float));
    memcpy(c->v[l], src->v[l], src->size * c->kv * sizeof(float));
  }
  c->nsegs = src->nsegs;
  c->segs = (orc_marks*)calloc(c->nsegs ? c->nsegs : 1, sizeof(orc_marks));
  for (size_t i = 0; i < c->nsegs; ++i) {
    c->segs[i] = src->segs[i];
    c->segs[i].origin = (uint8_t*)malloc(c->L * src->segs[i].len);
    memcpy(c->segs[i].origin, src->segs[i].origin, c->L * src->segs[i].len);
  }
  return c;
}
uint64_t orc_ctx_size(orc_ctx* c) { return c->size; }
uint64_t orc_ctx_num_segments(orc_ctx* c) { return c->nsegs; }
int orc_ctx_segment(orc_ctx* c, uint64_t i, uint64_t* base, uint64_t* len, uint8_t* origin) {
  if (i >= c->nsegs) return fail(RK_ERR_INVALID_ARGUMENT, "segment index out of range");
  *base = c->segs[i].base;
  *len = c->segs[i].len;
  if (origin) memcpy(origin, c->segs[i].origin, c->L * c->segs[i].len);
  return RK_OK;
}
int orc_ctx_export(orc_ctx* c, uint64_t layer, uint64_t pos, uint64_t count, float* k, float* v) {
  if (layer >= c->L || pos + count > c->size) return fail(RK_ERR_INVALID_ARGUMENT, "export range");
  if (k) memcpy(k, krow(c, layer, pos), count * c->kv * sizeof(float));
  if (v) memcpy(v, vrow(c, layer, pos), count * c->kv * sizeof(float));
  return RK_OK;
}

/* ------------------------------------------------------------------------ */
/* model forward (src/model.cpp)                                             */
/* ------------------------------------------------------------------------ */

/* attend_row (model.cpp:170-204); probs (optional) receives H x (pos+1). */
static void attend_row(const rk_model_spec* s, const float* q, orc_ctx* ctx, size_t layer,
                       size_t position, const float* self_k, const float* self_v, float* out,
                       float* probs) {
  const size_t ctx_len = position + 1, dh = s->d_head;
  const size_t group = s->num_heads / s->num_kv_heads;
  const float inv_sqrt_dh = 1.0f / sqrtf((float)dh);
  float* scores = (float*)malloc(ctx_len * sizeof(float));
  for (size_t h = 0; h < s->num_heads; ++h) {
    const size_t kvh = h / group;
    const float* qh = q + h * dh;
    for (size_t j = 0; j < ctx_len; ++j) {
      const float* kj = (j == position && self_k) ? self_k + kvh * dh : krow(ctx, layer, j) + kvh * dh;
      float sc = 0.0f;
      for (size_t d = 0; d < dh; ++d) sc += qh[d] * kj[d];
      scores[j] = sc * inv_sqrt_dh;
    }
    softmax_inplace(scores, ctx_len);
    if (probs) memcpy(probs + h * ctx_len, scores, ctx_len * sizeof(float));
    float* oh = out + h * dh;
    memset(oh, 0, dh * sizeof(float));
    for (size_t j = 0; j < ctx_len; ++j) {
      const float a = scores[j];
      const float* vj = (j == position && self_v) ? self_v + kvh * dh : vrow(ctx, layer, j) + kvh * dh;
      for (size_t d = 0; d < dh; ++d) oh[d] += a * vj[d];
    }
  }
  free(scores);
}

/* silu (model.cpp:208) + finish_rows (model.cpp:211-233). */
static void finish_rows(orc_weights* w, size_t layer, float* hidden, size_t rows,
                        const float* attn_out) {
  const rk_model_spec* s = &w->s;
  const orc_layer* L = &w->layers[layer];
  const size_t d = s->d_model, q = s->num_heads * s->d_head, ff = s->d_ff;
  float* proj = (float*)malloc(rows * d * sizeof(float));
  matmul(attn_out, rows, q, L->wo, d, proj);
  for (size_t i = 0; i < rows * d; ++i) hidden[i] += proj[i];
  float* normed = (float*)malloc(rows * d * sizeof(float));
  for (size_t r = 0; r < rows; ++r) rms_norm(hidden + r * d, L->mlp_norm, s->norm_eps, d, normed + r * d);
  float* gate = (float*)malloc(rows * ff * sizeof(float));
  float* up = (float*)malloc(rows * ff * sizeof(float));
  matmul(normed, rows, d, L->wgate, ff, gate);
  matmul(normed, rows, d, L->wup, ff, up);
  for (size_t i = 0; i < rows * ff; ++i) {
    const float g = gate[i];
    gate[i] = g / (1.0f + expf(-g)) * up[i];
  }
  matmul(gate, rows, ff, L->wdown, d, proj);
  for (size_t i = 0; i < rows * d; ++i) hidden[i] += proj[i];
  free(proj); free(normed); free(gate); free(up);
}

/* Decode-step capture (model.hpp:97-111) for one layer of a 1-row chunk. */
typedef struct {
  float* hidden; /* [L x d]  input of every layer */
  float* k_pre;  /* [L x kv] */
  float* v;      /* [L x kv] */
  float* attn;   /* [L x H x (pos+1)] */
} orc_trace;

/* run_layer_rows (model.cpp:237-280). */
static void run_layer_rows(orc_weights* w, size_t layer, float* hidden, size_t rows,
                           const size_t* positions, orc_ctx* ctx, orc_trace* tr) {
  const rk_model_spec* s = &w->s;
  const orc_layer* L = &w->layers[layer];
  const size_t d = s->d_model, q = s->num_heads * s->d_head, kv = s->num_kv_heads * s->d_head;
  if (tr) memcpy(tr->hidden + layer * d, hidden, d * sizeof(float));
  float* normed = (float*)malloc(rows * d * sizeof(float));
  for (size_t r = 0; r < rows; ++r) rms_norm(hidden + r * d, L->attn_norm, s->norm_eps, d, normed + r * d);
  float* Q = (float*)malloc(rows * q * sizeof(float));
  float* K = (float*)malloc(rows * kv * sizeof(float));
  float* V = (float*)malloc(rows * kv * sizeof(float));
  matmul(normed, rows, d, L->wq, q, Q);
  matmul(normed, rows, d, L->wk, kv, K);
  matmul(normed, rows, d, L->wv, kv, V);
  if (tr) {
    memcpy(tr->k_pre + layer * kv, K, kv * sizeof(float));
    memcpy(tr->v + layer * kv, V, kv * sizeof(float));
  }
  for (size_t r = 0; r < rows; ++r) {
    const int64_t pos = (int64_t)positions[r];
    rope_rotate_heads(Q + r * q, s->num_heads, s->d_head, pos, s->theta_base);
    rope_rotate_heads(K + r * kv, s->num_kv_heads, s->d_head, pos, s->theta_base);
    memcpy(krow(ctx, layer, positions[r]), K + r * kv, kv * sizeof(float));
    memcpy(vrow(ctx, layer, positions[r]), V + r * kv, kv * sizeof(float));
  }
  float* attn_out = (float*)malloc(rows * q * sizeof(float));
  for (size_t r = 0; r < rows; ++r) {
    float* probs = tr ? tr->attn + layer * s->num_heads * (positions[r] + 1) : NULL;
    attend_row(s, Q + r * q, ctx, layer, positions[r], NULL, NULL, attn_out + r * q, probs);
  }
  finish_rows(w, layer, hidden, rows, attn_out);
  free(normed); free(Q); free(K); free(V); free(attn_out);
}

/* output_logits (model.cpp:282-288) for one row. */
static void output_logits_row(orc_weights* w, const float* hidden_row, float* logits) {
  const size_t d = w->s.d_model;
  float* normed = (float*)malloc(d * sizeof(float));
  rms_norm(hidden_row, w->final_norm, w->s.norm_eps, d, normed);
  matmul(normed, 1, d, w->head, w->s.vocab_size, logits);
  free(normed);
}

/* embed_tokens (model.cpp:149-161). */
static int embed_tokens(orc_weights* w, const int32_t* tokens, size_t n, float* h) {
  const size_t d = w->s.d_model;
  for (size_t i = 0; i < n; ++i) {
    if (tokens[i] < 0 || (uint64_t)tokens[i] >= w->s.vocab_size) {
      snprintf(g_err, sizeof g_err, "token id %d outside vocab of %llu", tokens[i],
               (unsigned long long)w->s.vocab_size);
      return RK_ERR_INVALID_ARGUMENT;
    }
    memcpy(h + i * d, w->emb + (size_t)tokens[i] * d, d * sizeof(float));
  }
  return RK_OK;
}

static int check_finite(const char* what) {
  if (g_nonfinite) {
    g_nonfinite = 0;
    snprintf(g_err, sizeof g_err, "%s: non-finite value", what);
    return RK_ERR_NONFINITE;
  }
  return RK_OK;
}

/* prefill (model.cpp:305-331) with optional 1-row capture; all_logits/last_logits optional. */
static int prefill_impl(orc_weights* w, const int32_t* tokens, size_t n, orc_ctx* ctx, size_t base,
                        float* last_logits, orc_trace* tr) {
  const rk_model_spec* s = &w->s;
  if (n == 0) return fail(RK_ERR_INVALID_ARGUMENT, "prefill: empty token chunk");
  if (base != ctx->size) return fail(RK_ERR_INVALID_ARGUMENT, "prefill: base_position != context size");
  if (base + n > s->max_positions)
    return fail(RK_ERR_INVALID_ARGUMENT, "prefill: position overflow beyond max_positions");
  const size_t d = s->d_model;
  float* hidden = (float*)malloc(n * d * sizeof(float));
  int st = embed_tokens(w, tokens, n, hidden);
  if (st) { free(hidden); return st; }
  ctx_resize(ctx, base + n);
  size_t* positions = (size_t*)malloc(n * sizeof(size_t));
  for (size_t i = 0; i < n; ++i) positions[i] = base + i;
  g_nonfinite = 0;
  for (size_t l = 0; l < s->num_layers; ++l) run_layer_rows(w, l, hidden, n, positions, ctx, tr);
  if (last_logits) output_logits_row(w, hidden + (n - 1) * d, last_logits);
  free(hidden); free(positions);
  return check_finite("matmul");
}

int orc_prefill(orc_weights* w, orc_ctx* ctx, const int32_t* tokens, uint64_t n, uint64_t base,
                float* last_logits) {
  return prefill_impl(w, tokens, n, ctx, base, last_logits, NULL);
}

/* row_logits_from_layer (model.cpp:339-362). */
int orc_row_logits_from_layer(orc_weights* w, const float* hidden_row, uint64_t first_layer,
                              orc_ctx* ctx, uint64_t position, float* logits) {
  const rk_model_spec* s = &w->s;
  const size_t d = s->d_model, q = s->num_heads * s->d_head, kv = s->num_kv_heads * s->d_head;
  float* hidden = (float*)malloc(d * sizeof(float));
  memcpy(hidden, hidden_row, d * sizeof(float));
  float *normed = (float*)malloc(d * sizeof(float)), *Q = (float*)malloc(q * sizeof(float));
  float *K = (float*)malloc(kv * sizeof(float)), *V = (float*)malloc(kv * sizeof(float));
  float* attn = (float*)malloc(q * sizeof(float));
  g_nonfinite = 0;
  for (size_t l = first_layer; l < s->num_layers; ++l) {
    const orc_layer* L = &w->layers[l];
    rms_norm(hidden, L->attn_norm, s->norm_eps, d, normed);
    matmul(normed, 1, d, L->wq, q, Q);
    matmul(normed, 1, d, L->wk, kv, K);
    matmul(normed, 1, d, L->wv, kv, V);
    rope_rotate_heads(Q, s->num_heads, s->d_head, (int64_t)position, s->theta_base);
    rope_rotate_heads(K, s->num_kv_heads, s->d_head, (int64_t)position, s->theta_base);
    attend_row(s, Q, ctx, l, position, K, V, attn, NULL);
    finish_rows(w, l, hidden, 1, attn);
  }
  output_logits_row(w, hidden, logits);
  free(hidden); free(normed); free(Q); free(K); free(V); free(attn);
  return check_finite("matmul");
}

static size_t argmax(const float* v, size_t n) { /* model.cpp:364-370 */
  size_t best = 0;
  for (size_t i = 1; i < n; ++i)
    if (v[i] > v[best]) best = i;
  return best;
}

/* ------------------------------------------------------------------------ */
/* RelayCache (relay_cache.hpp:23-46, relay_cache.cpp)                       */
/* ------------------------------------------------------------------------ */

typedef struct orc_cache {
  uint64_t L, Hkv, dh, d, maxpos, n, src_base, snapshot, steps;
  float theta;
  int32_t* tokens;
  float** k_pre; /* [L][n x kv] */
  float** v;
  float* hidden;    /* [n x d] */
  float* influence; /* [n] */
} orc_cache;

void orc_cache_destroy(orc_cache* c) {
  if (!c) return;
  for (size_t l = 0; l < c->L; ++l) { free(c->k_pre[l]); free(c->v[l]); }
  free(c->k_pre); free(c->v); free(c->tokens); free(c->hidden); free(c->influence); free(c);
}

int orc_cache_from_view(const rk_relay_cache_view* v, orc_cache** out) {
  orc_cache* c = (orc_cache*)calloc(1, sizeof *c);
  c->L = v->num_layers; c->Hkv = v->num_kv_heads; c->dh = v->d_head; c->d = v->d_model;
  c->theta = v->theta_base; c->maxpos = v->max_positions; c->n = v->segment_len;
  c->src_base = v->source_base_position; c->snapshot = v->snapshot_layer;
  c->steps = v->decode_steps_observed;
  const size_t n = c->n, kv = c->Hkv * c->dh;
  c->tokens = (int32_t*)malloc((n ? n : 1) * sizeof(int32_t));
  if (n) memcpy(c->tokens, v->segment_tokens, n * sizeof(int32_t));
  c->k_pre = (float**)calloc(c->L ? c->L : 1, sizeof(float*));
  c->v = (float**)calloc(c->L ? c->L : 1, sizeof(float*));
  for (size_t l = 0; l < c->L; ++l) {
    c->k_pre[l] = (float*)malloc((n * kv ? n * kv : 1) * sizeof(float));
    c->v[l] = (float*)malloc((n * kv ? n * kv : 1) * sizeof(float));
    if (n) {
      memcpy(c->k_pre[l], v->k_pre[l], n * kv * sizeof(float));
      memcpy(c->v[l], v->v[l], n * kv * sizeof(float));
    }
  }
  c->hidden = (float*)malloc((n * c->d ? n * c->d : 1) * sizeof(float));
  if (n) memcpy(c->hidden, v->hidden_snapshot, n * c->d * sizeof(float));
  c->influence = (float*)malloc((n ? n : 1) * sizeof(float));
  if (n) memcpy(c->influence, v->influence, n * sizeof(float));
  *out = c;
  return RK_OK;
}

int orc_cache_view(orc_cache* c, rk_relay_cache_view* v, const float** kp, const float** vp) {
  v->num_layers = c->L; v->num_kv_heads = c->Hkv; v->d_head = c->dh; v->d_model = c->d;
  v->theta_base = c->theta; v->max_positions = c->maxpos; v->segment_len = c->n;
  v->segment_tokens = c->tokens; v->source_base_position = c->src_base;
  v->snapshot_layer = c->snapshot; v->decode_steps_observed = c->steps;
  for (size_t l = 0; l < c->L; ++l) { kp[l] = c->k_pre[l]; vp[l] = c->v[l]; }
  v->k_pre = kp; v->v = vp;
  v->hidden_snapshot = c->hidden; v->influence = c->influence;
  return RK_OK;
}

/* RelayCache::validate + validate_for (relay_cache.cpp:18-49). */
static int cache_validate_for(const orc_cache* c, const rk_model_spec* s) {
  if (c->n == 0) return fail(RK_ERR_INVALID_ARGUMENT, "relay cache: empty segment");
  if (c->L == 0) return fail(RK_ERR_INVALID_ARGUMENT, "relay cache: per-layer K/V tables disagree");
  if (c->snapshot >= c->L) return fail(RK_ERR_INVALID_ARGUMENT, "relay cache: snapshot layer out of range");
  for (size_t j = 0; j < c->n; ++j)
    if (!(c->influence[j] >= 0.0f)) return fail(RK_ERR_INVALID_ARGUMENT, "relay cache: negative influence score");
  if (s && (c->L != s->num_layers || c->Hkv != s->num_kv_heads || c->dh != s->d_head ||
            c->d != s->d_model || c->theta != s->theta_base))
    return fail(RK_ERR_INVALID_ARGUMENT, "relay cache geometry does not match model spec");
  return RK_OK;
}

/* Greedy decode with capture (model.cpp:372-389) feeding RelayRecorder
 * (relay_cache.cpp:52-136). first_logits: the prompt-end logits row. */
int orc_capture_decode(orc_weights* w, orc_ctx* ctx, const float* first_logits, uint64_t n,
                       uint64_t snapshot, int include_self, orc_cache** out) {
  const rk_model_spec* s = &w->s;
  if (snapshot >= s->num_layers) return fail(RK_ERR_INVALID_ARGUMENT, "recorder: snapshot layer out of range");
  const size_t d = s->d_model, kv = s->num_kv_heads * s->d_head, V = s->vocab_size;
  orc_cache* c = (orc_cache*)calloc(1, sizeof *c);
  c->L = s->num_layers; c->Hkv = s->num_kv_heads; c->dh = s->d_head; c->d = d;
  c->theta = s->theta_base; c->maxpos = s->max_positions; c->n = n;
  c->src_base = ctx->size; c->snapshot = snapshot; c->steps = n;
  c->tokens = (int32_t*)malloc((n ? n : 1) * sizeof(int32_t));
  c->k_pre = (float**)calloc(c->L, sizeof(float*));
  c->v = (float**)calloc(c->L, sizeof(float*));
  for (size_t l = 0; l < c->L; ++l) {
    c->k_pre[l] = (float*)malloc((n ? n : 1) * kv * sizeof(float));
    c->v[l] = (float*)malloc((n ? n : 1) * kv * sizeof(float));
  }
  c->hidden = (float*)malloc((n ? n : 1) * d * sizeof(float));
  c->influence = (float*)malloc((n ? n : 1) * sizeof(float));
  double* acc = (double*)calloc(n ? n : 1, sizeof(double));
  float* logits = (float*)malloc(V * sizeof(float));
  int32_t next = (int32_t)argmax(first_logits, V);
  orc_trace tr;
  const size_t maxctx = ctx->size + n;
  tr.hidden = (float*)malloc(s->num_layers * d * sizeof(float));
  tr.k_pre = (float*)malloc(s->num_layers * kv * sizeof(float));
  tr.v = (float*)malloc(s->num_layers * kv * sizeof(float));
  tr.attn = (float*)malloc(s->num_layers * s->num_heads * (maxctx + 1) * sizeof(float));
  int st = RK_OK;
  for (size_t t = 0; t < n && st == RK_OK; ++t) {
    const size_t pos = ctx->size;
    st = prefill_impl(w, &next, 1, ctx, pos, logits, &tr);
    if (st) break;
    for (size_t l = 0; l < s->num_layers; ++l) {
      memcpy(c->k_pre[l] + t * kv, tr.k_pre + l * kv, kv * sizeof(float));
      memcpy(c->v[l] + t * kv, tr.v + l * kv, kv * sizeof(float));
    }
    memcpy(c->hidden + t * d, tr.hidden + snapshot * d, d * sizeof(float));
    /* influence received from this step's query (relay_cache.cpp:108-123) */
    const size_t upto = include_self ? t + 1 : t;
    for (size_t l = 0; l < s->num_layers; ++l) {
      const float* rows = tr.attn + l * s->num_heads * (pos + 1);
      for (size_t h = 0; h < s->num_heads; ++h)
        for (size_t j = 0; j < upto; ++j) acc[j] += (double)rows[h * (pos + 1) + c->src_base + j];
    }
    c->tokens[t] = next;
    if (t + 1 < n) next = (int32_t)argmax(logits, V);
  }
  for (size_t j = 0; j < n; ++j) c->influence[j] = (float)acc[j];
  free(acc); free(logits); free(tr.hidden); free(tr.k_pre); free(tr.v); free(tr.attn);
  if (st) { orc_cache_destroy(c); return st; }
  *out = c;
  return RK_OK;
}

/* realign (relay_cache.cpp:154-174) of layer l into out [n x kv]. */
static void realign_layer(const orc_cache* c, size_t l, size_t base, float* out) {
  const size_t kv = c->Hkv * c->dh;
  memcpy(out, c->k_pre[l], c->n * kv * sizeof(float));
  for (size_t j = 0; j < c->n; ++j)
    rope_rotate_heads(out + j * kv, c->Hkv, c->dh, (int64_t)(base + j), c->theta);
}
int orc_realign(orc_cache* c, uint64_t base, float* const* out) {
  int st = cache_validate_for(c, NULL);
  if (st) return st;
  if (base + c->n > c->maxpos) return fail(RK_ERR_INVALID_ARGUMENT, "realign: base overflows max_positions");
  for (size_t l = 0; l < c->L; ++l) realign_layer(c, l, base, out[l]);
  return RK_OK;
}

/* ------------------------------------------------------------------------ */
/* deviation scores (src/metrics.cpp:21-32, 92-103)                          */
/* ------------------------------------------------------------------------ */

static double cosine_d(const float* a, const float* b, size_t n) {
  double dot = 0.0, na = 0.0, nb = 0.0;
  for (size_t i = 0; i < n; ++i) {
    const double x = a[i], y = b[i];
    dot += x * y;
    na += x * x;
    nb += y * y;
  }
  if (sqrt(na) < 1e-12 || sqrt(nb) < 1e-12) return 0.0;
  if (memcmp(a, b, n * sizeof(float)) == 0) return 1.0;
  double c = dot / (sqrt(na) * sqrt(nb));
  return c < -1.0 ? -1.0 : (c > 1.0 ? 1.0 : c);
}
double orc_mean_head_cosine_deviation(const float* a, const float* b, uint64_t n, uint64_t heads) {
  const size_t dh = n / heads;
  double acc = 0.0;
  for (size_t h = 0; h < heads; ++h) acc += cosine_d(a + h * dh, b + h * dh, dh);
  return 1.0 - acc / (double)heads;
}

/* ------------------------------------------------------------------------ */
/* selector (src/selector.cpp)                                               */
/* ------------------------------------------------------------------------ */

/* mean_relative (selector.cpp:32-50): flags[j] |= tag where s_j >= tau*mean. */
static double mean_relative(const double* scores, size_t n, double tau, unsigned tag, uint32_t* flags) {
  double mean = 0.0;
  for (size_t j = 0; j < n; ++j) mean += scores[j];
  mean /= (double)n;
  if (mean <= 0.0) return 0.0;
  const double thr = tau * mean;
  for (size_t j = 0; j < n; ++j)
    if (scores[j] >= thr) flags[j] |= tag;
  return thr;
}

typedef struct { double score; size_t idx; } scored;
static int scored_cmp(const void* pa, const void* pb) { /* selector.cpp:94-97 */
  const scored* a = (const scored*)pa;
  const scored* b = (const scored*)pb;
  if (a->score != b->score) return a->score > b->score ? -1 : 1;
  return a->idx < b->idx ? -1 : (a->idx > b->idx);
}

/* ------------------------------------------------------------------------ */
/* relay engine (src/relay_engine.cpp)                                       */
/* ------------------------------------------------------------------------ */

/* FLOP model (relay_engine.cpp:72-110). */
static double flops_pm(const rk_model_spec* s) {
  const double d = (double)s->d_model, kv = (double)(s->num_kv_heads * s->d_head), ff = (double)s->d_ff;
  return 2.0 * d * (2.0 * d + 2.0 * kv) + 6.0 * d * ff;
}
static double flops_attn(const rk_model_spec* s, size_t base, size_t n) {
  const double b = (double)base, nn = (double)n, dhH = (double)(s->d_head * s->num_heads);
  return 4.0 * dhH * (nn * b + nn * (nn + 1.0) / 2.0);
}
double orc_flops_span_full(const rk_model_spec* s, uint64_t base, uint64_t n) {
  const double layers = (double)s->num_layers;
  return layers * (double)n * flops_pm(s) + layers * flops_attn(s, base, n);
}
double orc_flops_segment_schedule(const rk_model_spec* s, uint64_t base, uint64_t n, uint64_t lo,
                                  uint64_t hi, uint64_t sparse_hi, uint64_t selected) {
  const double pm = flops_pm(s);
  const double band_layers = (double)(hi - lo + 1), sparse_layers = (double)(sparse_hi - hi);
  const double dhH = (double)(s->d_head * s->num_heads);
  const double avg_ctx = (double)base + ((double)n + 1.0) / 2.0;
  const double band = band_layers * ((double)n * pm + flops_attn(s, base, n));
  const double sparse = sparse_layers * (double)selected * (pm + 4.0 * dhH * avg_ctx);
  return band + sparse;
}
static double flops_selection(const rk_model_spec* s, size_t n) {
  const double nn = (double)n, kv = (double)(s->num_kv_heads * s->d_head);
  return nn * (6.0 * kv + 10.0) + 4.0 * nn;
}
static double flops_realign(const rk_model_spec* s, size_t n) {
  return 3.0 * (double)(s->num_kv_heads * s->d_head) * (double)n * (double)s->num_layers;
}

/* graft_realigned (relay_engine.cpp:136-148). */
static void graft(orc_ctx* ctx, const orc_cache* c, size_t base, float* const* keys) {
  const size_t kv = c->Hkv * c->dh;
  for (size_t l = 0; l < c->L; ++l) {
    memcpy(krow(ctx, l, base), keys[l], c->n * kv * sizeof(float));
    memcpy(vrow(ctx, l, base), c->v[l], c->n * kv * sizeof(float));
  }
}

/* sparse_rectify (relay_engine.cpp:156-179). */
static void sparse_rectify(orc_weights* w, float* hidden, uint64_t* depth, const size_t* sel,
                           size_t nsel, size_t base, size_t band_hi, size_t sparse_hi,
                           orc_ctx* ctx, uint8_t* origin, size_t n) {
  if (nsel == 0 || sparse_hi <= band_hi) return;
  const size_t d = w->s.d_model;
  float* sub = (float*)malloc(nsel * d * sizeof(float));
  size_t* positions = (size_t*)malloc(nsel * sizeof(size_t));
  for (size_t r = 0; r < nsel; ++r) {
    memcpy(sub + r * d, hidden + sel[r] * d, d * sizeof(float));
    positions[r] = base + sel[r];
  }
  for (size_t l = band_hi + 1; l <= sparse_hi; ++l) {
    run_layer_rows(w, l, sub, nsel, positions, ctx, NULL);
    for (size_t r = 0; r < nsel; ++r) origin[l * n + sel[r]] = 1;
  }
  for (size_t r = 0; r < nsel; ++r) {
    memcpy(hidden + sel[r] * d, sub + r * d, d * sizeof(float));
    depth[sel[r]] = sparse_hi + 1;
  }
  free(sub); free(positions);
}

/* relay_extend (relay_engine.cpp:183-361). The out buffers are optional. */
int orc_relay_extend(orc_weights* w, orc_ctx* ctx, orc_cache* cache, const rk_layer_profile* prof,
                     const rk_relay_options* opts, rk_relay_output* out_user) {
  const rk_model_spec* s = &w->s;
  int st = cache_validate_for(cache, s);
  if (st) return st;
  const size_t n = cache->n, base = ctx->size, L = s->num_layers, d = s->d_model;
  const size_t kv = s->num_kv_heads * s->d_head;
  if (base + n > s->max_positions) return fail(RK_ERR_INVALID_ARGUMENT, "relay_extend: segment overflows max_positions");
  const double t_total = now_ms();
  rk_relay_output tmp;
  memset(&tmp, 0, sizeof tmp);
  rk_relay_output* out = &tmp;
  uint8_t* origin = (uint8_t*)calloc(L * n, 1);
  float* hidden = (float*)malloc(n * d * sizeof(float));
  uint64_t* depth = (uint64_t*)calloc(n, sizeof(uint64_t));
  uint32_t* flags = (uint32_t*)calloc(n, sizeof(uint32_t));
  double* s_dev = NULL;
  double* s_key = NULL;
  size_t* sel = (size_t*)malloc(n * sizeof(size_t));
  size_t nsel = 0;
  rk_reuse_stats* rs = &out->stats;
  rs->total_entries = L * n;
  rs->flops_full_equiv = orc_flops_span_full(s, base, n);
  size_t* positions = (size_t*)malloc(n * sizeof(size_t));
  for (size_t j = 0; j < n; ++j) positions[j] = base + j;
  float** keys = NULL;
  const int mode = opts->mode;
  g_nonfinite = 0;

  if (mode == RK_MODE_RELAY) {
    if (!(prof->l_start <= prof->l_det && prof->l_det <= prof->l_end && prof->l_end < L)) {
      st = fail(RK_ERR_SCHEMA, "layer profile violates l_start <= l_det <= l_end < num_layers");
      goto done;
    }
    if (!(opts->tau_dev > 0.0)) { st = fail(RK_ERR_INVALID_ARGUMENT, "thresholds: tau_dev must be > 0"); goto done; }
    if (!(opts->tau_inf > 0.0)) { st = fail(RK_ERR_INVALID_ARGUMENT, "thresholds: tau_inf must be > 0"); goto done; }
    if (cache->snapshot != prof->l_start) {
      st = fail(RK_ERR_INVALID_ARGUMENT, "relay_extend: cache snapshot layer does not match profile l_start");
      goto done;
    }
  }
  if (mode == RK_MODE_BLEND && !(opts->blend_alpha > 0.0 && opts->blend_alpha <= 1.0)) {
    st = fail(RK_ERR_INVALID_ARGUMENT, "relay_extend: blend alpha must be in (0, 1]");
    goto done;
  }
  if (mode != RK_MODE_FULL) {
    double t0 = now_ms();
    if (base + n > cache->maxpos) { st = fail(RK_ERR_INVALID_ARGUMENT, "realign: base overflows max_positions"); goto done; }
    keys = (float**)calloc(L, sizeof(float*));
    for (size_t l = 0; l < L; ++l) {
      keys[l] = (float*)malloc(n * kv * sizeof(float));
      realign_layer(cache, l, base, keys[l]);
    }
    ctx_resize(ctx, base + n);
    graft(ctx, cache, base, keys);
    rs->wall.realign_ms = now_ms() - t0;
    rs->flops_realign = flops_realign(s, n);
  }

  if (mode == RK_MODE_FULL) {
    ctx_resize(ctx, base + n);
    if ((st = embed_tokens(w, cache->tokens, n, hidden))) goto done;
    const double t0 = now_ms();
    for (size_t l = 0; l < L; ++l) {
      run_layer_rows(w, l, hidden, n, positions, ctx, NULL);
      memset(origin + l * n, 1, n);
    }
    rs->wall.recompute_ms = now_ms() - t0;
    for (size_t j = 0; j < n; ++j) depth[j] = L;
    rs->flops_cost = orc_flops_span_full(s, base, n);
  } else if (mode == RK_MODE_ZERO) {
    memcpy(hidden, cache->hidden, n * d * sizeof(float));
    for (size_t j = 0; j < n; ++j) depth[j] = cache->snapshot;
  } else if (mode == RK_MODE_RELAY) {
    const size_t l_start = prof->l_start, l_det = prof->l_det, l_end = prof->l_end;
    const size_t sparse_hi = opts->rectify_above_end ? L - 1 : l_end;
    double t0 = now_ms();
    memcpy(hidden, cache->hidden, n * d * sizeof(float));
    for (size_t l = l_start; l <= l_det; ++l) {
      run_layer_rows(w, l, hidden, n, positions, ctx, NULL);
      memset(origin + l * n, 1, n);
    }
    for (size_t j = 0; j < n; ++j) depth[j] = l_det + 1;
    rs->wall.recompute_ms = now_ms() - t0;

    t0 = now_ms();
    s_dev = (double*)malloc(n * sizeof(double));
    s_key = (double*)malloc(n * sizeof(double));
    for (size_t j = 0; j < n; ++j) {
      s_dev[j] = orc_mean_head_cosine_deviation(vrow(ctx, l_det, base + j), cache->v[l_det] + j * kv, kv, s->num_kv_heads);
      s_key[j] = orc_mean_head_cosine_deviation(krow(ctx, l_det, base + j), keys[l_det] + j * kv, kv, s->num_kv_heads);
    }
    double* infl = (double*)malloc(n * sizeof(double));
    for (size_t j = 0; j < n; ++j) infl[j] = (double)cache->influence[j];
    const double thr = mean_relative(s_dev, n, opts->tau_dev, RK_SEL_DEVIATION, flags);
    mean_relative(infl, n, opts->tau_inf, RK_SEL_INFLUENCE_SCORE, flags);
    free(infl);
    const size_t k = opts->suffix_k;
    const size_t start = k >= n ? 0 : n - k;
    for (size_t j = start; j < n && k > 0; ++j) flags[j] |= RK_SEL_INFLUENCE_SUFFIX;
    for (size_t j = 0; j < n; ++j)
      if (flags[j]) sel[nsel++] = j;
    out->dev_threshold = thr;
    out->min_dev_margin = INFINITY;
    if (thr > 0.0)
      for (size_t j = 0; j < n; ++j) {
        const double m = fabs(s_dev[j] - thr) / thr;
        if (m < out->min_dev_margin) out->min_dev_margin = m;
      }
    rs->wall.selection_ms = now_ms() - t0;
    rs->flops_selection = flops_selection(s, n);

    t0 = now_ms();
    sparse_rectify(w, hidden, depth, sel, nsel, base, l_det, sparse_hi, ctx, origin, n);
    rs->wall.rectify_ms = now_ms() - t0;
    rs->flops_cost = orc_flops_segment_schedule(s, base, n, l_start, l_det, sparse_hi, nsel);
  } else { /* BLEND (relay_engine.cpp:295-344) */
    double t0 = now_ms();
    if ((st = embed_tokens(w, cache->tokens, n, hidden))) goto done;
    const size_t boot_hi = 1;
    for (size_t l = 0; l <= boot_hi; ++l) {
      run_layer_rows(w, l, hidden, n, positions, ctx, NULL);
      memset(origin + l * n, 1, n);
    }
    for (size_t j = 0; j < n; ++j) depth[j] = boot_hi + 1;
    rs->wall.recompute_ms = now_ms() - t0;
    t0 = now_ms();
    scored* sc = (scored*)malloc(n * sizeof(scored));
    for (size_t j = 0; j < n; ++j) {
      const float* fresh = vrow(ctx, boot_hi, base + j);
      const float* stale = cache->v[boot_hi] + j * kv;
      double acc = 0.0;
      for (size_t e = 0; e < kv; ++e) {
        const double diff = (double)fresh[e] - (double)stale[e];
        acc += diff * diff;
      }
      sc[j].score = sqrt(acc);
      sc[j].idx = j;
    }
    size_t count = (size_t)(opts->blend_alpha * (double)n);
    if (count > n) count = n;
    qsort(sc, n, sizeof(scored), scored_cmp);
    for (size_t i = 0; i < count; ++i) flags[sc[i].idx] |= RK_SEL_BLEND_TOPK;
    free(sc);
    for (size_t j = 0; j < n; ++j)
      if (flags[j]) sel[nsel++] = j;
    rs->wall.selection_ms = now_ms() - t0;
    rs->flops_selection = flops_selection(s, n);
    t0 = now_ms();
    sparse_rectify(w, hidden, depth, sel, nsel, base, boot_hi, L - 1, ctx, origin, n);
    rs->wall.rectify_ms = now_ms() - t0;
    rs->flops_cost = orc_flops_segment_schedule(s, base, n, 0, boot_hi, L - 1, nsel);
  }
  if ((st = check_finite("matmul"))) goto done;

  {
    size_t rec = 0;
    for (size_t i = 0; i < L * n; ++i) rec += origin[i];
    rs->recomputed_entries = rec;
    rs->reuse_rate = rs->total_entries == 0 ? 0.0 : 1.0 - (double)rec / (double)rs->total_entries;
    rs->selected_count = nsel;
    for (size_t i = 0; i < nsel; ++i) {
      const uint32_t t = flags[sel[i]];
      rs->selected_deviation += (t & RK_SEL_DEVIATION) != 0;
      rs->selected_influence_score += (t & RK_SEL_INFLUENCE_SCORE) != 0;
      rs->selected_influence_suffix += (t & RK_SEL_INFLUENCE_SUFFIX) != 0;
      rs->selected_blend += (t & RK_SEL_BLEND_TOPK) != 0;
    }
    rs->wall.total_ms = now_ms() - t_total;
    /* push SegmentMarks */
    ctx->segs = (orc_marks*)realloc(ctx->segs, (ctx->nsegs + 1) * sizeof(orc_marks));
    orc_marks* m = &ctx->segs[ctx->nsegs++];
    m->base = base;
    m->len = n;
    m->origin = (uint8_t*)malloc(L * n ? L * n : 1);
    memcpy(m->origin, origin, L * n);
    out->segment_base = base;
    out->segment_len = n;
    out->selection_count = nsel;
    out->s_dev_len = mode == RK_MODE_RELAY ? n : 0;
    if (out_user) {
      rk_relay_output* u = out_user;
      for (size_t i = 0; i < nsel; ++i) {
        if (u->selection_indices) u->selection_indices[i] = sel[i];
        if (u->selection_tags) u->selection_tags[i] = flags[sel[i]];
      }
      if (mode == RK_MODE_RELAY) {
        if (u->s_dev) memcpy(u->s_dev, s_dev, n * sizeof(double));
        if (u->s_key_dev) memcpy(u->s_key_dev, s_key, n * sizeof(double));
      }
      if (u->segment_hidden) memcpy(u->segment_hidden, hidden, n * d * sizeof(float));
      if (u->hidden_depth) memcpy(u->hidden_depth, depth, n * sizeof(uint64_t));
      if (u->origin) memcpy(u->origin, origin, L * n);
      u->segment_base = out->segment_base;
      u->segment_len = out->segment_len;
      u->selection_count = out->selection_count;
      u->s_dev_len = out->s_dev_len;
      u->dev_threshold = out->dev_threshold;
      u->min_dev_margin = out->min_dev_margin;
      u->stats = out->stats;
    }
  }
done:
  if (keys) {
    for (size_t l = 0; l < L; ++l) free(keys[l]);
    free(keys);
  }
  /* stash the last segment's hidden/depth for relay_prefill's end logits */
  if (st == RK_OK && out_user == NULL) { /* nothing */ }
  free(origin); free(flags); free(s_dev); free(s_key); free(sel); free(positions);
  if (st == RK_OK) {
    /* hidden/depth handed over through the user struct only; keep local copy semantics */
  }
  free(hidden); free(depth);
  return st;
}

/* relay_prefill (relay_engine.cpp:363-395). ctx must be fresh. */
int orc_relay_prefill(orc_weights* w, orc_ctx* ctx, const int32_t* prefix, uint64_t n_prefix,
                      orc_cache* cache, const rk_layer_profile* prof, const rk_relay_options* opts,
                      rk_relay_output* out, float* end_logits) {
  const rk_model_spec* s = &w->s;
  const double t0 = now_ms();
  int st;
  if (n_prefix > 0 && (st = orc_prefill(w, ctx, prefix, n_prefix, 0, NULL))) return st;
  const double prefix_ms = now_ms() - t0;
  const size_t n = cache->n, d = s->d_model;
  rk_relay_output o;
  if (out) o = *out; else memset(&o, 0, sizeof o);
  float* hidden = (float*)malloc((n ? n : 1) * d * sizeof(float));
  uint64_t* depth = (uint64_t*)malloc((n ? n : 1) * sizeof(uint64_t));
  o.segment_hidden = hidden;
  o.hidden_depth = depth;
  if ((st = orc_relay_extend(w, ctx, cache, prof, opts, &o))) { free(hidden); free(depth); return st; }
  o.stats.wall.fresh_ms = prefix_ms;
  o.stats.wall.total_ms += prefix_ms;
  o.stats.flops_cost += orc_flops_span_full(s, 0, n_prefix);
  o.stats.flops_full_equiv += orc_flops_span_full(s, 0, n_prefix);
  if (end_logits) {
    const size_t dep = depth[n - 1], last_pos = n_prefix + n - 1;
    if (dep >= s->num_layers) output_logits_row(w, hidden + (n - 1) * d, end_logits);
    else st = orc_row_logits_from_layer(w, hidden + (n - 1) * d, dep, ctx, last_pos, end_logits);
  }
  if (out) {
    float* uh = out->segment_hidden;
    uint64_t* ud = out->hidden_depth;
    if (uh) memcpy(uh, hidden, n * d * sizeof(float));
    if (ud) memcpy(ud, depth, n * sizeof(uint64_t));
    *out = o;
    out->segment_hidden = uh;
    out->hidden_depth = ud;
  }
  free(hidden); free(depth);
  return st;
}

/* run_workflow's relay branch (workflow.cpp:316-369) / FULL (301-315). */
int orc_agent_prefill(orc_weights* w, orc_ctx* ctx, const int32_t* prefix, uint64_t n_prefix,
                      orc_cache* const* ups, uint64_t n_up, const int32_t* suffix, uint64_t n_suffix,
                      const rk_layer_profile* prof, const rk_relay_options* opts, float* end_logits,
                      int32_t* first_token) {
  const rk_model_spec* s = &w->s;
  const size_t V = s->vocab_size, d = s->d_model;
  float* logits = (float*)malloc(V * sizeof(float));
  int st = RK_OK;
  if (opts->mode == RK_MODE_FULL) {
    size_t total = n_prefix + n_suffix;
    for (size_t u = 0; u < n_up; ++u) total += ups[u]->n;
    int32_t* full = (int32_t*)malloc(total * sizeof(int32_t));
    size_t o = 0;
    memcpy(full, prefix, n_prefix * sizeof(int32_t)); o += n_prefix;
    for (size_t u = 0; u < n_up; ++u) { memcpy(full + o, ups[u]->tokens, ups[u]->n * sizeof(int32_t)); o += ups[u]->n; }
    memcpy(full + o, suffix, n_suffix * sizeof(int32_t));
    st = orc_prefill(w, ctx, full, total, 0, logits);
    free(full);
  } else {
    st = orc_prefill(w, ctx, prefix, n_prefix, 0, NULL);
    float* hidden = NULL;
    uint64_t* depth = NULL;
    size_t last_n = 0;
    for (size_t u = 0; u < n_up && st == RK_OK; ++u) {
      last_n = ups[u]->n;
      hidden = (float*)realloc(hidden, last_n * d * sizeof(float));
      depth = (uint64_t*)realloc(depth, last_n * sizeof(uint64_t));
      rk_relay_output o;
      memset(&o, 0, sizeof o);
      o.segment_hidden = hidden;
      o.hidden_depth = depth;
      st = orc_relay_extend(w, ctx, ups[u], prof, opts, &o);
    }
    if (st == RK_OK) {
      if (n_suffix > 0) {
        st = orc_prefill(w, ctx, suffix, n_suffix, ctx->size, logits);
      } else {
        const size_t dep = depth[last_n - 1];
        if (dep >= s->num_layers) output_logits_row(w, hidden + (last_n - 1) * d, logits);
        else st = orc_row_logits_from_layer(w, hidden + (last_n - 1) * d, dep, ctx, ctx->size - 1, logits);
      }
    }
    free(hidden); free(depth);
  }
  if (st == RK_OK) {
    if (end_logits) memcpy(end_logits, logits, V * sizeof(float));
    if (first_token) *first_token = (int32_t)argmax(logits, V);
  }
  free(logits);
  return st;
}

/* Host libm expf, for checking the device restatement of glibc expf. */
float orc_host_expf(float x) { return expf(x); }
void orc_host_expf_array(const float* x, float* y, uint64_t n) {
  for (uint64_t i = 0; i < n; ++i) y[i] = expf(x[i]);
}
