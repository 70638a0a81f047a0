// rnntsim_cuda.hpp — C++ drop-in for the reference decoder interface.
//
// Same names and signatures as /root/reference/proj/include/rnntsim/
// decoders.hpp:56-130, in namespace rnntsim::cuda, running the B200 decoder
// behind the C ABI in include/rnntg.h.  A caller switches
//
//     rnntsim::greedy_decode_sync_free(engine, model, x, out_len, ms)
// to  rnntsim::cuda::greedy_decode_sync_free(engine, model, x, out_len, ms)
//
// and gets identical Hypotheses on the fp32 path (ties below the documented
// margin excepted).  build_decode_graph returns a reference CapturedDecoder
// whose bind_inputs / read_hypotheses closures drive the CUDA decoder, so the
// reference's own rnntsim::replay_decode also works on it unchanged.
//
// Errors: rnntg status codes are rethrown as the reference exception classes
// (errors.hpp:23-85).  Models: rnntsim::NeuralModel is recognised directly;
// any other DecoderModel (e.g. an LSTM prediction network) must also derive
// from CudaWeightSource to export its weights.  Models are immutable (as in
// the reference) and are uploaded once per model object.
#pragma once

#include <memory>
#include <vector>

#include "rnntg.h"
#include "rnntsim/decoders.hpp"
#include "rnntsim/engine.hpp"
#include "rnntsim/model.hpp"
#include "rnntsim/tensor.hpp"

namespace rnntsim {
namespace cuda {

/// Weight export for DecoderModel implementations other than NeuralModel:
/// dims plus host pointers in the order documented in rnntg.h
/// (rnntg_model_create).
class CudaWeightSource {
 public:
  virtual ~CudaWeightSource() = default;
  virtual rnntg_dims cuda_dims() const = 0;
  virtual std::vector<const float*> cuda_weights() const = 0;
};

/// Executor used by the functions below (default: the tensor-core persistent
/// kernel; shapes it does not take fall back to the FFMA persistent kernel,
/// then to the CUDA graph).
void set_executor(rnntg_exec exec);
rnntg_exec executor();

Hypotheses greedy_decode_sync_free(Engine& engine, const DecoderModel& model, const Tensor& x,
                                   const Tensor& out_len, int max_symbols);
Hypotheses label_looping_decode(Engine& engine, const DecoderModel& model, const Tensor& x,
                                const Tensor& out_len, int max_symbols);
Hypotheses tdt_label_looping_decode(Engine& engine, const DecoderModel& model, const Tensor& x,
                                    const Tensor& out_len, int max_symbols);
CapturedDecoder build_decode_graph(Engine& engine, const DecoderModel& model, DecodeAlgo algo,
                                   int batch, int max_frames, int max_symbols);
Hypotheses replay_decode(CapturedDecoder& captured, const Tensor& x, const Tensor& out_len);
/// replay_decode plus the reference's TimingReport (engine.hpp:119-128) of
/// this decode, measured on the device instead of simulated: CUPTI kernel
/// activity gives span_us (first kernel start -> last kernel end),
/// device_busy_us (union of kernel intervals, graph kernel nodes counted
/// individually), idle_fraction = 1 - busy/span and num_kernels; the host
/// wall time of the launch call is host_busy_us; num_syncs / num_graph_launches
/// come from the library's host counters (rnntg_host_counts).  The report feeds
/// the reference's compare_runs / speedup_table_csv (analysis.cpp:112-154)
/// unchanged.  Throws StateError for an uninitialized capture.
Hypotheses replay_decode_timed(CapturedDecoder& captured, const Tensor& x, const Tensor& out_len,
                               TimingReport* report);
/// Joint-step evaluations of the last CUDA decode issued with this engine.
int64_t decode_joint_evals(const Engine& engine);

/// Release the device copies of every uploaded model.
void release_models();

}  // namespace cuda
}  // namespace rnntsim
