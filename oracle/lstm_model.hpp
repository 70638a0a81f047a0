// lstm_model.hpp — the LSTM prediction network as a reference DecoderModel.
//
// TEST INFRASTRUCTURE ONLY (oracle extension).
// The reference ships only a 1-layer tanh RNN (model.hpp:42-44, SPEC.md:201
// "LSTM not required"), while every BASELINE config names a 2-layer LSTM.
// The DecoderModel interface explicitly allows new models (model.hpp:89-126),
// so this class plugs an L-layer LSTM into the UNMODIFIED reference decoders.
// Its joint delegates to the reference's own rnntsim::joint / joint_tdt
// (model.cpp:178-213) on the top layer's h; the cell uses reference tensor
// ops with the same operation order as oracle/rnnt_oracle.c:
//   gates = (x @ W_ih + h @ W_hh) + b   (order i, f, g, o)
//   c' = f*c + i*g ; h' = o*tanh(c') ; sigma(x) = 1/(1+exp(-x))
// State layout [h_0, c_0, ..., h_{L-1}, c_{L-1}] (one vector per row).
#pragma once

#include <cmath>
#include <utility>
#include <vector>

#include "rnnt_oracle.h"  // orc_dims layout only
#include "rnntsim/model.hpp"
#include "rnntsim/tensor.hpp"

namespace oracle {

inline rnntsim::Tensor tensor_from(const float* p, int64_t rows, int64_t cols) {
  std::vector<float> v(p, p + rows * cols);
  return rnntsim::Tensor::from_floats(std::move(v), {rows, cols}, /*checked=*/false);
}

inline float sigmoid_ref(float x) { return 1.0f / (1.0f + std::exp(-x)); }

class LstmModel : public rnntsim::DecoderModel {
 public:
  LstmModel(const orc_dims& d, const float* const* p) : d_(d) {
    using rnntsim::Tensor;
    const int64_t V1 = d.vocab + 1, E = d.embed, H = d.hidden;
    jp_.dims.vocab = d.vocab;
    jp_.dims.embed = d.embed;
    jp_.dims.hidden = d.hidden;
    jp_.dims.joint = d.joint;
    jp_.dims.feature = d.feature;
    jp_.dims.durations.assign(d.durations, d.durations + d.num_durations);
    jp_.dims.validate();
    jp_.embedding = tensor_from(p[0], V1, E);
    for (int l = 0; l < d.layers; ++l) {
      const int64_t in = l == 0 ? E : H;
      w_ih_.push_back(tensor_from(p[1 + 3 * l], in, 4 * H));
      w_hh_.push_back(tensor_from(p[2 + 3 * l], H, 4 * H));
      bias_.push_back(tensor_from(p[3 + 3 * l], 1, 4 * H));
    }
    const int base = 1 + 3 * d.layers;
    jp_.enc_proj = tensor_from(p[base], d.feature, d.joint);
    jp_.pred_proj = tensor_from(p[base + 1], H, d.joint);
    jp_.out_proj = tensor_from(p[base + 2], d.joint, V1);
    if (d.num_durations > 0) jp_.dur_proj = tensor_from(p[base + 3], d.joint, d.num_durations);
  }

  const orc_dims& dims() const { return d_; }
  const rnntsim::RnntParams& joint_params() const { return jp_; }
  const rnntsim::Tensor& w_ih(int l) const { return w_ih_[l]; }
  const rnntsim::Tensor& w_hh(int l) const { return w_hh_[l]; }
  const rnntsim::Tensor& bias(int l) const { return bias_[l]; }

  int vocab_size() const override { return d_.vocab; }
  int state_width() const override { return 2 * d_.layers * d_.hidden; }
  int feature_dim() const override { return d_.feature; }
  const std::vector<int32_t>& durations() const override { return jp_.dims.durations; }

  void run_prediction(const rnntsim::Tensor& last_label, const rnntsim::Tensor& hidden,
                      rnntsim::Tensor& hidden_prime) const override {
    using rnntsim::Dtype;
    using rnntsim::Tensor;
    const int64_t B = last_label.numel(), H = d_.hidden, W = state_width();
    Tensor out(Dtype::Float32, {B, W});
    Tensor x(Dtype::Float32, {B, d_.embed});
    rnntsim::embedding_lookup_into(jp_.embedding, last_label, x);
    for (int l = 0; l < d_.layers; ++l) {
      Tensor h(Dtype::Float32, {B, H}), c(Dtype::Float32, {B, H});
      for (int64_t b = 0; b < B; ++b) {
        std::copy_n(&hidden.f32()[b * W + 2 * l * H], H, &h.f32()[b * H]);
        std::copy_n(&hidden.f32()[b * W + (2 * l + 1) * H], H, &c.f32()[b * H]);
      }
      Tensor ih(Dtype::Float32, {B, 4 * H}), hh(Dtype::Float32, {B, 4 * H});
      rnntsim::matmul_into(x, w_ih_[l], ih);
      rnntsim::matmul_into(h, w_hh_[l], hh);
      Tensor hn(Dtype::Float32, {B, H});
      auto pi = ih.f32();
      auto ph = hh.f32();
      auto pb = bias_[l].f32();
      for (int64_t b = 0; b < B; ++b) {
        for (int64_t j = 0; j < H; ++j) {
          const int64_t r = b * 4 * H;
          const float gi = (pi[r + j] + ph[r + j]) + pb[j];
          const float gf = (pi[r + H + j] + ph[r + H + j]) + pb[H + j];
          const float gg = (pi[r + 2 * H + j] + ph[r + 2 * H + j]) + pb[2 * H + j];
          const float go = (pi[r + 3 * H + j] + ph[r + 3 * H + j]) + pb[3 * H + j];
          const float i_ = sigmoid_ref(gi), f_ = sigmoid_ref(gf);
          const float g_ = std::tanh(gg), o_ = sigmoid_ref(go);
          const float cn = f_ * c.f32()[b * H + j] + i_ * g_;
          out.f32()[b * W + (2 * l + 1) * H + j] = cn;
          const float hv = o_ * std::tanh(cn);
          out.f32()[b * W + 2 * l * H + j] = hv;
          hn.f32()[b * H + j] = hv;
        }
      }
      x = std::move(hn);
    }
    hidden_prime.assign(out);
  }

  rnntsim::Tensor top(const rnntsim::Tensor& g) const {
    const int64_t B = g.dim(0), H = d_.hidden, W = state_width();
    rnntsim::Tensor t(rnntsim::Dtype::Float32, {B, H});
    for (int64_t b = 0; b < B; ++b)
      std::copy_n(&g.f32()[b * W + 2 * (d_.layers - 1) * H], H, &t.f32()[b * H]);
    return t;
  }

  void run_joint(const rnntsim::Tensor& f, const rnntsim::Tensor& g,
                 rnntsim::Tensor& logp) const override {
    logp.assign(rnntsim::joint(jp_, f, top(g)));
  }
  void run_joint_tdt(const rnntsim::Tensor& f, const rnntsim::Tensor& g,
                     rnntsim::Tensor& token_logp, rnntsim::Tensor& dur_logp) const override {
    auto [tok, dur] = rnntsim::joint_tdt(jp_, f, top(g));
    token_logp.assign(tok);
    dur_logp.assign(dur);
  }

 private:
  orc_dims d_;
  rnntsim::RnntParams jp_;
  std::vector<rnntsim::Tensor> w_ih_, w_hh_, bias_;
};

}  // namespace oracle
