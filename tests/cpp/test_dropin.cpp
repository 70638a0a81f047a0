// test_dropin.cpp — the reference's own acceptance checks (tests/acceptance.cpp
// criteria 1-2, test_decoders.cpp) run through the C++ drop-in
// rnntsim::cuda::* (include/rnntsim_cuda.hpp) against the UNMODIFIED
// reference decoders, in one binary linked with the reference library
// (oracle/_ref) and the CUDA library.  Prints PASS/FAIL lines; exit code =
// number of failures.  Needs a B200.
#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "decode_test_util.hpp"
#include "lstm_model.hpp"
#include "rnntsim/analysis.hpp"
#include "rnntsim/decoders.hpp"
#include "rnntsim/errors.hpp"
#include "rnntsim_cuda.hpp"
#include "cuda_lstm.hpp"

using namespace rnntsim;

namespace {

int g_fail = 0;

void report(const char* name, bool ok, const std::string& detail) {
  std::printf("%s: %s  %s\n", name, ok ? "PASS" : "FAIL", detail.c_str());
  if (!ok) ++g_fail;
}

// Tokens and frames exact; scores within 1e-4 relative (denominator
// max(|ref|, 1e-3)); the GPU fp32 arithmetic differs from the reference's
// sequential order at the ulp level (SURVEY.md §8c comparator).
bool same(const Hypotheses& a, const Hypotheses& b, double* max_rel) {
  if (a.size() != b.size()) return false;
  for (size_t i = 0; i < a.size(); ++i) {
    if (a[i].tokens != b[i].tokens || a[i].frames != b[i].frames) return false;
    for (size_t j = 0; j < a[i].scores.size(); ++j) {
      const double r = std::fabs((double)a[i].scores[j] - b[i].scores[j]) /
                       std::max(std::fabs((double)b[i].scores[j]), 1e-3);
      *max_rel = std::max(*max_rel, r);
      if (r > 1e-4) return false;
    }
  }
  return true;
}

// Scripted models: tokens, frames exact; a planted decision scores
// 10 - lse with lse = 10 + log(1 + V e^-10) ~ 10.0007 in fp32 on both sides,
// so one rounding step of lse (ulp(10) = 9.5e-7) separates two correct
// summation orders; scores are compared to 4e-6 absolute.
bool same_scripted(const Hypotheses& a, const Hypotheses& b) {
  if (a.size() != b.size()) return false;
  for (size_t i = 0; i < a.size(); ++i) {
    if (a[i].tokens != b[i].tokens || a[i].frames != b[i].frames) return false;
    for (size_t j = 0; j < a[i].scores.size(); ++j)
      if (std::fabs((double)a[i].scores[j] - b[i].scores[j]) > 4e-6) return false;
  }
  return true;
}

}  // namespace

int main() {
  if (rnntg_device_count() < 1) {
    std::printf("no CUDA device\n");
    return 1;
  }
  for (rnntg_exec ex : {RNNTG_EXEC_GRAPH, RNNTG_EXEC_PERSISTENT, RNNTG_EXEC_TENSOR, RNNTG_EXEC_HOSTLOOP}) {
    cuda::set_executor(ex);
    const char* en = ex == RNNTG_EXEC_GRAPH ? "graph" : ex == RNNTG_EXEC_PERSISTENT ? "persistent"
                     : ex == RNNTG_EXEC_TENSOR ? "tensor" : "hostloop";
    // criterion 1 analogue: 200 random configs x 4 drop-in decoders
    int mism = 0;
    double rel = 0.0;
    for (uint64_t seed = 1; seed <= 200; ++seed) {
      const testutil::RandomCase c = testutil::make_random_case(seed, false);
      const Hypotheses expect = testutil::oracle_batch(c.model, c.x, c.out_len, c.max_symbols, false);
      Engine eng;
      std::vector<Hypotheses> got;
      got.push_back(cuda::greedy_decode_sync_free(eng, c.model, c.x, c.out_len, c.max_symbols));
      got.push_back(cuda::label_looping_decode(eng, c.model, c.x, c.out_len, c.max_symbols));
      CapturedDecoder cap = cuda::build_decode_graph(eng, c.model, DecodeAlgo::FrameSync,
                                                     (int)c.x.dim(0), (int)c.x.dim(1), c.max_symbols);
      got.push_back(cuda::replay_decode(cap, c.x, c.out_len));
      // the reference's own replay_decode drives the CUDA CapturedDecoder unchanged
      got.push_back(rnntsim::replay_decode(cap, c.x, c.out_len));
      for (const auto& g : got)
        if (!same(g, expect, &rel)) ++mism;
    }
    report((std::string("dropin exactness ") + en).c_str(), mism == 0,
           "200 configs x 4 decoders, " + std::to_string(mism) + " mismatches, max score rel " +
               std::to_string(rel));
    // criterion 2 analogue: TDT seeds 1000..1199
    mism = 0;
    rel = 0.0;
    for (uint64_t seed = 1000; seed < 1200; ++seed) {
      const testutil::RandomCase c = testutil::make_random_case(seed, true);
      Engine eng;
      const Hypotheses got = cuda::tdt_label_looping_decode(eng, c.model, c.x, c.out_len, c.max_symbols);
      if (!same(got, testutil::oracle_batch(c.model, c.x, c.out_len, c.max_symbols, true), &rel)) ++mism;
    }
    report((std::string("dropin tdt ") + en).c_str(), mism == 0,
           "200 configs, " + std::to_string(mism) + " mismatches");
    // 2-layer LSTM (C2 dims, short) through the unmodified reference decoders vs the drop-in
    {
      orc_dims d{};
      d.vocab = 1024;
      d.embed = d.hidden = 640;
      d.layers = 2;
      d.cell = ORC_CELL_LSTM;
      d.joint = 640;
      d.feature = 1024;
      std::vector<std::vector<float>> w(static_cast<size_t>(orc_num_params(&d)));
      std::vector<float*> wp;
      for (int i = 0; i < orc_num_params(&d); ++i) {
        int64_t r, cc;
        orc_param_size(&d, i, &r, &cc);
        w[i].resize(static_cast<size_t>(r * cc));
        wp.push_back(w[i].data());
      }
      orc_init_params(1, &d, wp.data());
      CudaLstm model(d, w);
      Tensor x(Dtype::Float32, {3, 6, 1024});
      orc_fill_uniform(2, -1.0f, 1.0f, x.f32().data(), x.numel());
      const Tensor lens = Tensor::from_ints({6, 4, 6}, {3});
      Engine e1, e2;
      const Hypotheses ref = rnntsim::greedy_decode_sync_free(e1, model, x, lens, 5);
      const Hypotheses got = cuda::greedy_decode_sync_free(e2, model, x, lens, 5);
      rel = 0.0;
      report((std::string("dropin lstm-2x640 ") + en).c_str(), same(got, ref, &rel),
             "joint evals " + std::to_string(cuda::decode_joint_evals(e2)) + ", max score rel " +
                 std::to_string(rel));
    }
    // error mapping (errors.hpp)
    {
      const testutil::RandomCase c = testutil::make_random_case(5, false);
      Engine eng;
      bool ok = true;
      try {
        cuda::greedy_decode_sync_free(eng, c.model, c.x, c.out_len, 0);
        ok = false;
      } catch (const ValueError&) {
      }
      try {
        Tensor bad = Tensor::from_ints(std::vector<int32_t>((size_t)c.x.dim(0), 999), {c.x.dim(0)});
        cuda::greedy_decode_sync_free(eng, c.model, c.x, bad, 2);
        ok = false;
      } catch (const DimensionError&) {
      }
      try {
        cuda::tdt_label_looping_decode(eng, c.model, c.x, c.out_len, 2);
        ok = false;
      } catch (const StateError&) {
      }
      report((std::string("dropin errors ") + en).c_str(), ok,
             "ValueError / DimensionError / StateError as in errors.hpp");
    }
  }
  // §8(f)4: the reference's planted-trace schedule tests on the GPU schedules
  // through a device ScriptedModel (test_decoders.cpp:57-80, 107-133,
  // 292-309, 404-431; acceptance.cpp criterion 8), against the reference's
  // own decoders on the CPU.
  for (rnntg_exec ex : {RNNTG_EXEC_GRAPH, RNNTG_EXEC_HOSTLOOP, RNNTG_EXEC_TENSOR}) {
    cuda::set_executor(ex);  // TENSOR: scripted models fall back to the graph executor
    const std::string en = ex == RNNTG_EXEC_GRAPH ? "graph" : ex == RNNTG_EXEC_HOSTLOOP ? "hostloop" : "default";
    auto adversarial_pair = [](int frames, int ms, int vocab) {
      ScriptedModel::LabelTable table(2, std::vector<std::vector<int32_t>>(frames));
      for (int b = 0; b < 2; ++b)
        for (int t = 0; t < frames; ++t)
          if (t % 2 == b % 2)
            for (int j = 0; j < ms; ++j) table[b][t].push_back((t * ms + j) % vocab);
      return ScriptedModel(vocab, ms, std::move(table));
    };
    bool ok = true;
    std::string why;
    auto expect = [&](bool c, const std::string& what) {
      if (!c && ok) why = what;
      ok = ok && c;
    };
    {  // planted script, empty script, emission cap
      ScriptedModel m1(8, 5, {{{3}, {}, {5, 6}}});
      ScriptedModel m2(8, 5, {{{}, {}}});
      ScriptedModel m3(16, 5, {{{1, 2, 3, 4, 5, 6, 7}, {9}}});
      Engine e1, e2, e3, r1;
      const Hypotheses h1 = cuda::greedy_decode_sync_free(e1, m1, m1.make_features(), Tensor::from_ints({3}, {1}), 5);
      const Hypotheses h2 = cuda::greedy_decode_sync_free(e2, m2, m2.make_features(), Tensor::from_ints({2}, {1}), 5);
      const Hypotheses h3 = cuda::greedy_decode_sync_free(e3, m3, m3.make_features(), Tensor::from_ints({2}, {1}), 5);
      expect(h1[0].tokens == std::vector<int32_t>{3, 5, 6} && h1[0].frames == std::vector<int32_t>{0, 2, 2}, "planted");
      expect(h2[0].tokens.empty(), "empty script");
      expect(h3[0].tokens == std::vector<int32_t>{1, 2, 3, 4, 5, 9} &&
                 h3[0].frames == std::vector<int32_t>{0, 0, 0, 0, 0, 1},
             "emission cap");
      expect(same_scripted(h1, rnntsim::greedy_decode_sync_free(r1, m1, m1.make_features(), Tensor::from_ints({3}, {1}), 5)),
             "planted vs reference");
    }
    {  // adversarial even/odd pair: FS 20 joint evaluations, LL 12, identical hypotheses
      const ScriptedModel m = adversarial_pair(4, 5, 16);
      const Tensor x = m.make_features();
      const Tensor len = Tensor::from_ints({4, 4}, {2});
      Engine fs_e, ll_e, ref_e;
      const Hypotheses fs = cuda::greedy_decode_sync_free(fs_e, m, x, len, 5);
      const Hypotheses ll = cuda::label_looping_decode(ll_e, m, x, len, 5);
      const Hypotheses ref = rnntsim::greedy_decode_sync_free(ref_e, m, x, len, 5);
      auto show = [](const Hypotheses& h) {
        std::string o;
        for (const auto& y : h) {
          o += "[";
          for (size_t i = 0; i < y.tokens.size(); ++i)
            o += std::to_string(y.tokens[i]) + "@" + std::to_string(y.frames[i]) + " ";
          o += "]";
        }
        return o;
      };
      expect(same_scripted(fs, ref) && same_scripted(ll, ref),
             "adversarial pair vs reference: fs " + show(fs) + " ll " + show(ll) + " ref " + show(ref));
      expect(fs[0].frames == std::vector<int32_t>({0, 0, 0, 0, 0, 2, 2, 2, 2, 2}) &&
                 fs[1].frames == std::vector<int32_t>({1, 1, 1, 1, 1, 3, 3, 3, 3, 3}),
             "adversarial frames");
      // criterion 8: label looping does strictly less joint work.  The reference
      // counts 12 (one joint + a prediction for every row per iteration); the
      // device label loop is the nested blank-skipping form (SURVEY.md §8 a16:
      // joint-only inner iterations until no row awaits a decision, then the
      // acceptors' prediction), which spends one extra joint here: at frame 0
      // utterance 1 blanks while utterance 0 waits with its accepted label.
      expect(cuda::decode_joint_evals(fs_e) == 20 && cuda::decode_joint_evals(ll_e) == 13 &&
                 cuda::decode_joint_evals(ll_e) < cuda::decode_joint_evals(fs_e),
             "joint evals FS " + std::to_string(cuda::decode_joint_evals(fs_e)) + " LL " +
                 std::to_string(cuda::decode_joint_evals(ll_e)));
      for (DecodeAlgo algo : {DecodeAlgo::FrameSync, DecodeAlgo::LabelLoop}) {  // graph replay
        Engine eng;
        CapturedDecoder cap = cuda::build_decode_graph(eng, m, algo, 2, 4, 5);
        expect(same_scripted(cuda::replay_decode(cap, x, len), ref), "replay");
      }
    }
    {  // planted durations skip frames: tokens {1,2,3,4} at frames {0,0,2,5}
      ScriptedModel m(9, 3, {{{1, 2}, {}, {3}, {}, {}, {4}}}, {0, 1, 2, 3, 4},
                      {{{0, 2, 1}, {}, {3, 1}, {}, {}, {0, 1}}});
      const Tensor x = m.make_features();
      const Tensor len = Tensor::from_ints({6}, {1});
      Engine e, r;
      const Hypotheses got = cuda::tdt_label_looping_decode(e, m, x, len, 3);
      expect(got[0].tokens == std::vector<int32_t>({1, 2, 3, 4}) && got[0].frames == std::vector<int32_t>({0, 0, 2, 5}),
             "planted durations");
      expect(same_scripted(got, rnntsim::tdt_label_looping_decode(r, m, x, len, 3)), "durations vs reference");
    }
    report(("dropin scripted model (f)4 " + en).c_str(), ok,
           ok ? "planted / empty / cap / adversarial pair (FS 20 vs LL 13 joint evals; reference 20 vs 12) / durations {0,0,2,5}"
              : "failed: " + why);
  }
  // §8(f)3: the reference's TimingReport measured on the device
  // (cuda::replay_decode_timed, CUPTI) for each executor on a C2-dims batch,
  // through the reference's own compare_runs / speedup_table_csv
  // (analysis.cpp:112-154) against the sync-requiring host loop (Alg. 1).
  {
    orc_dims d{};
    d.vocab = 1024;
    d.embed = d.hidden = 640;
    d.layers = 2;
    d.cell = ORC_CELL_LSTM;
    d.joint = 640;
    d.feature = 1024;
    std::vector<std::vector<float>> w(static_cast<size_t>(orc_num_params(&d)));
    std::vector<float*> wp;
    for (int i = 0; i < orc_num_params(&d); ++i) {
      int64_t r, cc;
      orc_param_size(&d, i, &r, &cc);
      w[i].resize(static_cast<size_t>(r * cc));
      wp.push_back(w[i].data());
    }
    orc_init_params(1, &d, wp.data());
    CudaLstm model(d, w);
    const int B = 32, T = 40, ms = 5;
    Tensor x(Dtype::Float32, {B, T, 1024});
    orc_fill_uniform(2, -1.0f, 1.0f, x.f32().data(), x.numel());
    const Tensor lens = Tensor::from_ints(std::vector<int32_t>(B, T), {B});
    const double audio_s = B * T * 0.08;  // 80 ms encoder frames (8x subsampled 10 ms features)
    struct Run {
      const char* name;
      rnntg_exec ex;
      TimingReport rep;
      Hypotheses hyps;
    };
    std::vector<Run> runs = {{"sync-requiring host loop (Alg. 1)", RNNTG_EXEC_HOSTLOOP, {}, {}},
                             {"conditional-WHILE CUDA graph", RNNTG_EXEC_GRAPH, {}, {}},
                             {"FFMA persistent kernel", RNNTG_EXEC_PERSISTENT, {}, {}},
                             {"tcgen05 persistent kernel", RNNTG_EXEC_TENSOR, {}, {}}};
    bool ok = true;
    for (Run& r : runs) {
      cuda::set_executor(r.ex);
      Engine eng;
      CapturedDecoder cap = cuda::build_decode_graph(eng, model, DecodeAlgo::FrameSync, B, T, ms);
      cuda::replay_decode(cap, x, lens);  // warm-up
      r.hyps = cuda::replay_decode_timed(cap, x, lens, &r.rep);
      std::printf("timing %-36s %s\n", r.name, timing_report_json(r.rep).c_str());
      ok = ok && r.rep.span_us > 0.0 && r.rep.num_kernels > 0 && r.rep.device_busy_us <= r.rep.span_us * 1.0001;
    }
    const TimingReport& base = runs[0].rep;
    ok = ok && base.num_syncs > 2 * T;  // a flag readback per inner step
    // sync-free executors: only the read-back syncs (counts + stats), no per-step ones
    ok = ok && runs[1].rep.num_graph_launches == 1 && runs[1].rep.num_syncs <= 2;
    ok = ok && runs[3].rep.num_syncs <= 2 && runs[3].rep.idle_fraction < 0.1;
    std::vector<SpeedupTableRow> rows;
    rows.push_back({runs[0].name, rtfx(audio_s, base.span_us * 1e-6), 100.0, 0.0, 1.0, 1.0});
    for (size_t i = 1; i < runs.size(); ++i) {
      try {
        const SpeedupReport s = compare_runs(base, runs[0].hyps, runs[i].rep, runs[i].hyps, 0.0, audio_s);
        rows.push_back({runs[i].name, s.rtfx_after, 100.0 * s.decoder_fraction_after, s.wer_between,
                        s.overall_speedup, s.decoder_speedup});
        ok = ok && s.decoder_speedup > 1.0;
      } catch (const Error& e) {
        std::printf("compare_runs(%s): %s\n", runs[i].name, e.what());
        ok = false;
      }
    }
    std::printf("%s", speedup_table_csv(rows).c_str());
    report("dropin timing report (f)3", ok,
           "host-loop idle " + std::to_string(base.idle_fraction) + ", tensor idle " +
               std::to_string(runs[3].rep.idle_fraction) + ", tensor decoder speed-up " +
               std::to_string(base.span_us / runs[3].rep.span_us));
  }
  cuda::release_models();
  return g_fail;
}
