// cuda_lstm.hpp — oracle::LstmModel (the reference-decoder LSTM extension)
// exporting its weights to the CUDA drop-in (rnntsim::cuda::CudaWeightSource).
// Shared by the drop-in acceptance binary and tools/rnntg_cli.cpp.
#pragma once

#include <vector>

#include "lstm_model.hpp"
#include "rnntsim_cuda.hpp"

namespace rnntsim {

class CudaLstm : public oracle::LstmModel, public cuda::CudaWeightSource {
 public:
  CudaLstm(const orc_dims& d, std::vector<std::vector<float>> w)
      : oracle::LstmModel(d, ptrs(w).data()), d_(d), w_(std::move(w)) {}
  rnntg_dims cuda_dims() const override {
    rnntg_dims r{};
    r.vocab = d_.vocab;
    r.embed = d_.embed;
    r.hidden = d_.hidden;
    r.layers = d_.layers;
    r.cell = RNNTG_CELL_LSTM;
    r.joint = d_.joint;
    r.feature = d_.feature;
    r.num_durations = d_.num_durations;
    for (int i = 0; i < d_.num_durations; ++i) r.durations[i] = d_.durations[i];
    return r;
  }
  std::vector<const float*> cuda_weights() const override {
    std::vector<const float*> p;
    for (const auto& v : w_) p.push_back(v.data());
    return p;
  }

 private:
  static std::vector<const float*> ptrs(const std::vector<std::vector<float>>& w) {
    std::vector<const float*> p;
    for (const auto& v : w) p.push_back(v.data());
    return p;
  }
  orc_dims d_;
  std::vector<std::vector<float>> w_;
};

}  // namespace rnntsim
