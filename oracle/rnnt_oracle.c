/*
 * rnnt_oracle.c — CPU restatement of the reference greedy-decode path.
 *
 * TEST INFRASTRUCTURE ONLY (see rnnt_oracle.h).  Build with
 *   gcc -O2 -ffp-contract=off -fPIC -shared
 * so every float operation rounds exactly as the reference's
 * (/root/reference/proj/CMakeLists.txt:12-13 uses -ffp-contract=off).
 *
 * Each function cites the reference lines it restates.  The matmul loop is
 * interchanged (i,k,j) for speed; every output still accumulates its k terms
 * in ascending order with one rounding per add, so results are bit-identical
 * to matmul_into (tensor.cpp:237-258).
 */
#include "rnnt_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- Rng */
/* tensor.cpp:633-640 — splitmix64 */
uint64_t orc_rng_next(orc_rng* r) {
  uint64_t z = (r->state += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

/* tensor.cpp:642-645 */
float orc_rng_uniform(orc_rng* r, float lo, float hi) {
  const float u = (float)(orc_rng_next(r) >> 40) * 0x1.0p-24f;
  return lo + (hi - lo) * u;
}

/* tensor.cpp:650-653 */
int32_t orc_rng_uniform_int(orc_rng* r, int32_t n) {
  if (n <= 0) return 0;
  return (int32_t)(orc_rng_next(r) % (uint64_t)n);
}

void orc_fill_uniform(uint64_t seed, float lo, float hi, float* out, int64_t n) {
  orc_rng r = {seed};
  for (int64_t i = 0; i < n; ++i) out[i] = orc_rng_uniform(&r, lo, hi);
}

/* ---------------------------------------------------------------- dims */
/* model.cpp:65-79 (RnntDims::validate) + LSTM extension checks. */
int orc_validate_dims(const orc_dims* d) {
  if (d->vocab < 1 || d->embed < 1 || d->hidden < 1 || d->joint < 1 ||
      d->feature < 1)
    return -1;
  if (d->cell != ORC_CELL_TANH && d->cell != ORC_CELL_LSTM) return -1;
  if (d->layers < 1 || d->layers > ORC_MAX_LAYERS) return -1;
  if (d->cell == ORC_CELL_TANH && d->layers != 1) return -1;
  if (d->num_durations < 0 || d->num_durations > ORC_MAX_DURATIONS) return -1;
  if (d->num_durations > 0) {
    if (d->durations[0] != 0 && d->durations[0] != 1) return -1;
    for (int i = 1; i < d->num_durations; ++i)
      if (d->durations[i] <= d->durations[i - 1]) return -1;
  }
  return 0;
}

int orc_state_width(const orc_dims* d) {
  return d->cell == ORC_CELL_TANH ? d->hidden : 2 * d->layers * d->hidden;
}

int orc_num_params(const orc_dims* d) {
  const int head = d->num_durations > 0 ? 1 : 0;
  return 1 + 3 * d->layers + 3 + head;
}

int orc_param_size(const orc_dims* d, int i, int64_t* rows, int64_t* cols) {
  const int64_t v1 = d->vocab + 1, E = d->embed, H = d->hidden, J = d->joint,
                F = d->feature, D = d->num_durations;
  const int64_t G = d->cell == ORC_CELL_LSTM ? 4 * H : H;
  const int L = d->layers;
  if (i < 0 || i >= orc_num_params(d)) return -1;
  if (i == 0) { *rows = v1; *cols = E; return 0; }
  if (i <= 3 * L) {
    const int l = (i - 1) / 3, which = (i - 1) % 3;
    const int64_t in = l == 0 ? E : H;
    if (which == 0) { *rows = in; *cols = G; }
    else if (which == 1) { *rows = H; *cols = G; }
    else { *rows = 1; *cols = G; }
    return 0;
  }
  const int j = i - 1 - 3 * L;
  switch (j) {
    case 0: *rows = F; *cols = J; return 0;
    case 1: *rows = H; *cols = J; return 0;
    case 2: *rows = J; *cols = v1; return 0;
    case 3: *rows = J; *cols = D; return 0;
  }
  return -1;
}

/* model.cpp:81-108 — fixed fill order, U[-0.08,0.08).  The LSTM extension
 * keeps the same order with per-layer (w_ih, w_hh, bias) triples. */
int orc_init_params(uint64_t seed, const orc_dims* d, float* const* out) {
  if (orc_validate_dims(d)) return -1;
  orc_rng r = {seed};
  const int n = orc_num_params(d);
  for (int i = 0; i < n; ++i) {
    int64_t rows, cols;
    orc_param_size(d, i, &rows, &cols);
    const int64_t cnt = rows * cols;
    for (int64_t e = 0; e < cnt; ++e) out[i][e] = orc_rng_uniform(&r, -0.08f, 0.08f);
  }
  return 0;
}

/* ---------------------------------------------------------------- ops */
/* tensor.cpp:237-258: out[i,j] = sum_k a[i,k] b[k,j], k ascending, no FMA. */
static void matmul(const float* a, int64_t lda, const float* b, float* out,
                   int64_t m, int64_t k, int64_t n) {
  for (int64_t i = 0; i < m; ++i) {
    float* o = out + i * n;
    for (int64_t j = 0; j < n; ++j) o[j] = 0.0f;
    for (int64_t kk = 0; kk < k; ++kk) {
      const float av = a[i * lda + kk];
      const float* brow = b + kk * n;
      for (int64_t j = 0; j < n; ++j) o[j] += av * brow[j];
    }
  }
}

/* tensor.cpp:463-480 */
static void log_softmax_row(const float* row, float* out, int64_t n) {
  float m = row[0];
  for (int64_t j = 1; j < n; ++j) m = (m < row[j]) ? row[j] : m; /* std::max */
  float sum = 0.0f;
  for (int64_t j = 0; j < n; ++j) sum += expf(row[j] - m);
  const float lse = m + logf(sum);
  for (int64_t j = 0; j < n; ++j) out[j] = row[j] - lse;
}

/* tensor.cpp:268-312 (first strict max; lowest index wins ties), plus the
 * top-2 margin used by the divergence accounting. */
static int argmax_row(const float* a, int64_t n, float* best_v, float* margin) {
  int best = 0;
  float bv = a[0];
  for (int64_t j = 1; j < n; ++j)
    if (a[j] > bv) { bv = a[j]; best = (int)j; }
  float second = -INFINITY;
  for (int64_t j = 0; j < n; ++j)
    if (j != best && a[j] > second) second = a[j];
  *best_v = bv;
  if (margin) *margin = n > 1 ? bv - second : INFINITY;
  return best;
}

static float sigmoidf_ref(float x) { return 1.0f / (1.0f + expf(-x)); }

/* Parameter accessors. */
#define P_EMB(p) ((p)[0])
#define P_WIH(p, l) ((p)[1 + 3 * (l)])
#define P_WHH(p, l) ((p)[2 + 3 * (l)])
#define P_B(p, l) ((p)[3 + 3 * (l)])
#define P_ENC(p, d) ((p)[1 + 3 * (d)->layers])
#define P_PRED(p, d) ((p)[2 + 3 * (d)->layers])
#define P_OUT(p, d) ((p)[3 + 3 * (d)->layers])
#define P_DUR(p, d) ((p)[4 + 3 * (d)->layers])

/* tanh cell: model.cpp:163-176 + rnn_cell_into 39-51.
 * LSTM cell (extension): gates = (x@W_ih + h@W_hh) + b
 * in order i,f,g,o; c' = f*c + i*g; h' = o*tanh(c'); sigma = 1/(1+exp(-x)). */
void orc_prediction(const orc_dims* d, const float* const* p, int batch,
                    const int32_t* labels, const float* state,
                    float* state_out) {
  const int64_t H = d->hidden, E = d->embed, W = orc_state_width(d);
  const int64_t G = d->cell == ORC_CELL_LSTM ? 4 * H : H;
  float* ih = (float*)malloc(sizeof(float) * G);
  float* hh = (float*)malloc(sizeof(float) * G);
  float* x = (float*)malloc(sizeof(float) * (E > H ? E : H));
  for (int b = 0; b < batch; ++b) {
    const float* s = state + b * W;
    float* so = state_out + b * W;
    /* embedding_lookup_into (tensor.cpp:489-506); id range checked there. */
    int32_t id = labels[b];
    if (id < 0 || id > d->vocab) id = d->vocab; /* caller guarantees range */
    memcpy(x, P_EMB(p) + (int64_t)id * E, sizeof(float) * E);
    int64_t in = E;
    for (int l = 0; l < d->layers; ++l) {
      const float* h_l = d->cell == ORC_CELL_TANH ? s : s + 2 * l * H;
      matmul(x, in, P_WIH(p, l), ih, 1, in, G);
      matmul(h_l, H, P_WHH(p, l), hh, 1, H, G);
      const float* bias = P_B(p, l);
      if (d->cell == ORC_CELL_TANH) {
        for (int64_t j = 0; j < H; ++j) so[j] = tanhf(ih[j] + hh[j] + bias[j]);
      } else {
        const float* c_l = s + (2 * l + 1) * H;
        float* ho = so + 2 * l * H;
        float* co = so + (2 * l + 1) * H;
        for (int64_t j = 0; j < H; ++j) {
          const float gi = (ih[j] + hh[j]) + bias[j];
          const float gf = (ih[H + j] + hh[H + j]) + bias[H + j];
          const float gg = (ih[2 * H + j] + hh[2 * H + j]) + bias[2 * H + j];
          const float go = (ih[3 * H + j] + hh[3 * H + j]) + bias[3 * H + j];
          const float i_ = sigmoidf_ref(gi), f_ = sigmoidf_ref(gf);
          const float g_ = tanhf(gg), o_ = sigmoidf_ref(go);
          const float c = f_ * c_l[j] + i_ * g_;
          co[j] = c;
          ho[j] = o_ * tanhf(c);
        }
        memcpy(x, ho, sizeof(float) * H);
        in = H;
      }
    }
  }
  free(ih);
  free(hh);
  free(x);
}

/* model.cpp:178-213 (joint / joint_tdt). */
void orc_joint(const orc_dims* d, const float* const* p, int batch,
               const float* f, const float* g, int64_t g_stride, float* logp,
               float* dur_logp) {
  const int64_t J = d->joint, F = d->feature, H = d->hidden, V1 = d->vocab + 1,
                D = d->num_durations;
  float* fp = (float*)malloc(sizeof(float) * J);
  float* gp = (float*)malloc(sizeof(float) * J);
  float* trunk = (float*)malloc(sizeof(float) * J);
  float* logits = (float*)malloc(sizeof(float) * (V1 > D ? V1 : D));
  for (int b = 0; b < batch; ++b) {
    matmul(f + b * F, F, P_ENC(p, d), fp, 1, F, J);
    matmul(g + b * g_stride, H, P_PRED(p, d), gp, 1, H, J);
    for (int64_t j = 0; j < J; ++j) {
      const float s = fp[j] + gp[j];
      trunk[j] = (s < 0.0f) ? 0.0f : s; /* relu_add_into: std::max(s, 0) */
    }
    matmul(trunk, J, P_OUT(p, d), logits, 1, J, V1);
    log_softmax_row(logits, logp + b * V1, V1);
    if (dur_logp && D > 0) {
      matmul(trunk, J, P_DUR(p, d), logits, 1, J, D);
      log_softmax_row(logits, dur_logp + b * D, D);
    }
  }
  free(fp);
  free(gp);
  free(trunk);
  free(logits);
}

/* decoders.cpp:670-701 (tdt=0) and 703-755 (tdt=1). */
int orc_decode_utt(const orc_dims* d, const float* const* p,
                   const float* features, int frames, int out_len,
                   int max_symbols, int tdt, int32_t* tokens, int32_t* frm,
                   float* scores, int32_t* durs, int cap, orc_decision* dec,
                   int dcap, int* ndec, double* total) {
  (void)frames;
  const int64_t W = orc_state_width(d), F = d->feature, V1 = d->vocab + 1,
                D = d->num_durations;
  const int blank = d->vocab;
  const int64_t g_off = d->cell == ORC_CELL_TANH ? 0 : 2 * (d->layers - 1) * d->hidden;
  float* hidden = (float*)calloc((size_t)W, sizeof(float));
  float* h_prime = (float*)calloc((size_t)W, sizeof(float));
  float* logp = (float*)malloc(sizeof(float) * V1);
  float* dlogp = (float*)malloc(sizeof(float) * (D > 0 ? D : 1));
  int32_t last = blank;
  int n = 0, nd = 0;
  double tot = 0.0;
  if (!tdt) {
    for (int t = 0; t < out_len; ++t) {
      const float* f = features + (int64_t)t * F;
      for (int sym = 0; sym < max_symbols; ++sym) {
        orc_prediction(d, p, 1, &last, hidden, h_prime);
        orc_joint(d, p, 1, f, h_prime + g_off, W, logp, NULL);
        float v, margin;
        const int k = argmax_row(logp, V1, &v, &margin);
        if (dec && nd < dcap) {
          orc_decision r = {t, k, -1, 0, v, margin, 0.0f};
          dec[nd] = r;
        }
        ++nd;
        if (k == blank) break;
        if (n < cap) {
          if (tokens) tokens[n] = k;
          if (frm) frm[n] = t;
          if (scores) scores[n] = v;
          if (durs) durs[n] = 0;
        }
        ++n;
        last = k;
        memcpy(hidden, h_prime, sizeof(float) * W);
      }
    }
  } else {
    int t = 0, u = 0;
    while (t < out_len) {
      const float* f = features + (int64_t)t * F;
      orc_prediction(d, p, 1, &last, hidden, h_prime);
      orc_joint(d, p, 1, f, h_prime + g_off, W, logp, dlogp);
      float v, margin, dv, dmargin;
      const int k = argmax_row(logp, V1, &v, &margin);
      const int di = argmax_row(dlogp, D, &dv, &dmargin);
      const int dur = d->durations[di];
      if (dec && nd < dcap) {
        orc_decision r = {t, k, di, dur, v, margin, dmargin};
        dec[nd] = r;
      }
      ++nd;
      if (k != blank) {
        if (n < cap) {
          if (tokens) tokens[n] = k;
          if (frm) frm[n] = t;
          if (scores) scores[n] = v;
          if (durs) durs[n] = dur;
        }
        ++n;
        last = k;
        memcpy(hidden, h_prime, sizeof(float) * W);
        u += 1;
        if (dur > 0) {
          t += dur;
          u = 0;
        } else if (u == max_symbols) {
          t += 1;
          u = 0;
        }
      } else {
        t += dur > 1 ? dur : 1;
        u = 0;
      }
    }
  }
  /* decoders.cpp:699-700: total in double, emission order. */
  if (scores) {
    const int m = n < cap ? n : cap;
    for (int i = 0; i < m; ++i) tot += (double)scores[i];
  }
  if (ndec) *ndec = nd;
  if (total) *total = tot;
  free(hidden);
  free(h_prime);
  free(logp);
  free(dlogp);
  return n;
}

/* decode_test_util.hpp:38-59 */
uint64_t orc_random_case_header(uint64_t seed, int with_durations,
                                orc_dims* d, int* batch, int* frames,
                                int* max_symbols) {
  orc_rng r = {seed};
  memset(d, 0, sizeof(*d));
  d->vocab = 5 + orc_rng_uniform_int(&r, 26);
  d->embed = 4 + orc_rng_uniform_int(&r, 13);
  d->hidden = 4 + orc_rng_uniform_int(&r, 13);
  d->joint = 4 + orc_rng_uniform_int(&r, 13);
  d->feature = 4 + orc_rng_uniform_int(&r, 13);
  d->layers = 1;
  d->cell = ORC_CELL_TANH;
  if (with_durations) {
    d->num_durations = 5;
    for (int i = 0; i < 5; ++i) d->durations[i] = i;
  }
  *batch = 1 + orc_rng_uniform_int(&r, 8);
  *frames = 1 + orc_rng_uniform_int(&r, 20);
  *max_symbols = 1 + orc_rng_uniform_int(&r, 5);
  return seed * 7919 + 1;
}

void orc_random_case_inputs(uint64_t seed, float* x, int32_t* out_len) {
  orc_rng r = {seed};
  orc_dims d;
  memset(&d, 0, sizeof(d));
  for (int i = 0; i < 5; ++i) (void)orc_rng_next(&r); /* dims draws */
  const int batch = 1 + orc_rng_uniform_int(&r, 8);
  const int frames = 1 + orc_rng_uniform_int(&r, 20);
  (void)orc_rng_next(&r); /* max_symbols draw */
  /* feature width is the 5th draw; recompute it from a fresh stream */
  orc_rng r2 = {seed};
  for (int i = 0; i < 4; ++i) (void)orc_rng_next(&r2);
  const int feature = 4 + orc_rng_uniform_int(&r2, 13);
  const int64_t nx = (int64_t)batch * frames * feature;
  for (int64_t i = 0; i < nx; ++i) x[i] = orc_rng_uniform(&r, -1.0f, 1.0f);
  for (int b = 0; b < batch; ++b) out_len[b] = orc_rng_uniform_int(&r, frames + 1);
}
