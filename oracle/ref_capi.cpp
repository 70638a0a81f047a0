// ref_capi.cpp — C entry points over the UNMODIFIED reference decoders.
//
// TEST INFRASTRUCTURE ONLY.  Compiled (by oracle/Makefile) together with the
// reference sources where they lie under /root/reference/proj/src into
// oracle/_ref/librnntsim_ref.so.  Used by tests/ to pin the C restatement
// (oracle/rnnt_oracle.c) and by bench.py's CPU arms (cpu_baseline and
// --impl reference) to time the reference's own decoders on host cores.
//
// The one addition is `LstmModel` (oracle/lstm_model.hpp), a DecoderModel
// subclass implementing the LSTM prediction network the BASELINE configs
// name, plugged into the unmodified reference decoders.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <memory>
#include <thread>
#include <vector>

#include "decode_test_util.hpp"  // /root/reference/proj/tests (by include path)
#include "lstm_model.hpp"
#include "rnnt_oracle.h"         // orc_dims layout only
#include "rnntsim/decoders.hpp"
#include "rnntsim/engine.hpp"
#include "rnntsim/model.hpp"
#include "rnntsim/tensor.hpp"

using namespace rnntsim;

namespace {

using oracle::LstmModel;
using oracle::tensor_from;

struct RefModel {
  orc_dims d{};
  std::unique_ptr<DecoderModel> model;
};

std::unique_ptr<DecoderModel> make_model(const orc_dims& d, const float* const* p) {
  if (d.cell == ORC_CELL_LSTM) return std::make_unique<LstmModel>(d, p);
  RnntParams rp;
  rp.dims.vocab = d.vocab;
  rp.dims.embed = d.embed;
  rp.dims.hidden = d.hidden;
  rp.dims.joint = d.joint;
  rp.dims.feature = d.feature;
  rp.dims.durations.assign(d.durations, d.durations + d.num_durations);
  const int64_t V1 = d.vocab + 1;
  rp.embedding = tensor_from(p[0], V1, d.embed);
  rp.w_ih = tensor_from(p[1], d.embed, d.hidden);
  rp.w_hh = tensor_from(p[2], d.hidden, d.hidden);
  rp.bias = Tensor::from_floats(std::vector<float>(p[3], p[3] + d.hidden),
                                {d.hidden}, false);
  rp.enc_proj = tensor_from(p[4], d.feature, d.joint);
  rp.pred_proj = tensor_from(p[5], d.hidden, d.joint);
  rp.out_proj = tensor_from(p[6], d.joint, V1);
  if (d.num_durations > 0) rp.dur_proj = tensor_from(p[7], d.joint, d.num_durations);
  return std::make_unique<NeuralModel>(std::move(rp));
}

// algo: 0 scalar oracle per utterance (tdt flag picks the variant),
// 1 greedy_decode_baseline, 2 greedy_decode_sync_free, 3 FrameSync graph
// replay, 4 label_looping_decode, 5 LabelLoop graph replay,
// 6 tdt_label_looping_decode, 7 TdtLabelLoop graph replay.
Hypotheses run_algo(Engine& eng, const DecoderModel& m, int algo, const Tensor& x,
                    const Tensor& out_len, int ms) {
  const int B = static_cast<int>(x.dim(0)), T = static_cast<int>(x.dim(1));
  switch (algo) {
    case 0: return testutil::oracle_batch(m, x, out_len, ms, false);
    case 8: return testutil::oracle_batch(m, x, out_len, ms, true);
    case 1: return greedy_decode_baseline(eng, m, x, out_len, ms);
    case 2: return greedy_decode_sync_free(eng, m, x, out_len, ms);
    case 3: {
      CapturedDecoder c = build_decode_graph(eng, m, DecodeAlgo::FrameSync, B, T, ms);
      return replay_decode(c, x, out_len);
    }
    case 4: return label_looping_decode(eng, m, x, out_len, ms);
    case 5: {
      CapturedDecoder c = build_decode_graph(eng, m, DecodeAlgo::LabelLoop, B, T, ms);
      return replay_decode(c, x, out_len);
    }
    case 6: return tdt_label_looping_decode(eng, m, x, out_len, ms);
    case 7: {
      CapturedDecoder c =
          build_decode_graph(eng, m, DecodeAlgo::TdtLabelLoop, B, T, ms);
      return replay_decode(c, x, out_len);
    }
  }
  throw ValueError("unknown algo");
}

void store(const Hypotheses& h, int b0, int32_t* counts, int32_t* tokens,
           int32_t* frames, float* scores, double* totals, int cap) {
  for (size_t i = 0; i < h.size(); ++i) {
    const int b = b0 + static_cast<int>(i);
    const auto& y = h[i];
    const int n = static_cast<int>(y.tokens.size());
    counts[b] = n;
    totals[b] = y.total_score;
    for (int e = 0; e < n && e < cap; ++e) {
      tokens[static_cast<int64_t>(b) * cap + e] = y.tokens[e];
      frames[static_cast<int64_t>(b) * cap + e] = y.frames[e];
      scores[static_cast<int64_t>(b) * cap + e] = y.scores[e];
    }
  }
}

thread_local std::string g_err;

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// Runs one of the reference decoders on make_random_case(seed) and writes
// the hypotheses into [batch, cap] arrays.  Returns batch (or -1).
int ref_random_case_decode(uint64_t seed, int with_dur, int algo, int32_t* counts,
                           int32_t* tokens, int32_t* frames, float* scores,
                           double* totals, int cap, int64_t* joint_evals) {
  try {
    const testutil::RandomCase c = testutil::make_random_case(seed, with_dur != 0);
    Engine eng;
    const Hypotheses h = run_algo(eng, c.model, algo, c.x, c.out_len, c.max_symbols);
    store(h, 0, counts, tokens, frames, scores, totals, cap);
    if (joint_evals) *joint_evals = decode_joint_evals(eng);
    return static_cast<int>(h.size());
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// Reference NeuralModel parameters for make_random_case(seed), in fill order.
int ref_random_case_params(uint64_t seed, int with_dur, float* const* out) {
  const testutil::RandomCase c = testutil::make_random_case(seed, with_dur != 0);
  const RnntParams& p = c.model.params();
  const Tensor* ts[] = {&p.embedding, &p.w_ih, &p.w_hh, &p.bias, &p.enc_proj,
                        &p.pred_proj, &p.out_proj, &p.dur_proj};
  const int n = with_dur ? 8 : 7;
  for (int i = 0; i < n; ++i)
    std::memcpy(out[i], ts[i]->f32().data(), ts[i]->numel() * sizeof(float));
  return n;
}

void* ref_model_create(const orc_dims* d, const float* const* params) {
  try {
    auto* m = new RefModel;
    m->d = *d;
    m->model = make_model(*d, params);
    return m;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void ref_model_destroy(void* h) { delete static_cast<RefModel*>(h); }

// Decodes x[B,T,F] with the chosen reference decoder, sharding utterances over
// `threads` std::threads (one Engine each; engine.hpp:136-138).  Returns 0 on
// success; *seconds gets the wall time of the decode calls only.
int ref_decode(void* h, int algo, const float* x, int B, int T,
               const int32_t* out_len, int ms, int threads, int32_t* counts,
               int32_t* tokens, int32_t* frames, float* scores, double* totals,
               int cap, double* seconds) {
  auto* m = static_cast<RefModel*>(h);
  const int F = m->d.feature;
  threads = std::max(1, std::min(threads, B));
  std::vector<Tensor> xs(threads), ls(threads);
  std::vector<int> b0(threads + 1);
  for (int i = 0; i <= threads; ++i) b0[i] = static_cast<int>((int64_t)B * i / threads);
  for (int i = 0; i < threads; ++i) {
    const int nb = b0[i + 1] - b0[i];
    std::vector<float> xv(x + (int64_t)b0[i] * T * F, x + (int64_t)b0[i + 1] * T * F);
    xs[i] = Tensor::from_floats(std::move(xv), {nb, T, F}, false);
    ls[i] = Tensor::from_ints(std::vector<int32_t>(out_len + b0[i], out_len + b0[i + 1]), {nb});
  }
  std::vector<Hypotheses> res(threads);
  std::vector<std::string> errs(threads);
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> pool;
  for (int i = 0; i < threads; ++i) {
    pool.emplace_back([&, i] {
      try {
        Engine eng;
        res[i] = run_algo(eng, *m->model, algo, xs[i], ls[i], ms);
      } catch (const std::exception& e) {
        errs[i] = e.what();
      }
    });
  }
  for (auto& t : pool) t.join();
  const auto t1 = std::chrono::steady_clock::now();
  if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
  for (int i = 0; i < threads; ++i) {
    if (!errs[i].empty()) {
      g_err = errs[i];
      return -1;
    }
    store(res[i], b0[i], counts, tokens, frames, scores, totals, cap);
  }
  return 0;
}

void ref_joint(void* h, int batch, const float* f, const float* g_state,
               float* logp, float* dur_logp) {
  auto* m = static_cast<RefModel*>(h);
  const int W = m->model->state_width(), F = m->d.feature;
  const int V1 = m->d.vocab + 1, D = m->d.num_durations;
  Tensor ft = tensor_from(f, batch, F), gt = tensor_from(g_state, batch, W);
  Tensor lp(Dtype::Float32, {batch, V1});
  if (dur_logp && D > 0) {
    Tensor dl(Dtype::Float32, {batch, D});
    m->model->run_joint_tdt(ft, gt, lp, dl);
    std::memcpy(dur_logp, dl.f32().data(), sizeof(float) * batch * D);
  } else {
    m->model->run_joint(ft, gt, lp);
  }
  std::memcpy(logp, lp.f32().data(), sizeof(float) * batch * V1);
}

void ref_prediction(void* h, int batch, const int32_t* labels,
                    const float* state, float* state_out) {
  auto* m = static_cast<RefModel*>(h);
  const int W = m->model->state_width();
  Tensor lt = Tensor::from_ints(std::vector<int32_t>(labels, labels + batch), {batch});
  Tensor st = tensor_from(state, batch, W), out(Dtype::Float32, {batch, W});
  m->model->run_prediction(lt, st, out);
  std::memcpy(state_out, out.f32().data(), sizeof(float) * batch * W);
}

}  // extern "C"
