// rnntg_cli.cpp — the reference CLI's decode route (cli.cpp:277-348, commands
// gen / decode / compare of tools/rnntsim_main.cpp) running the B200 decoder.
//
//   rnntg_cli gen --out DIR [--batch 8 --frames 32 --feature-dim 16 --vocab 16
//                            --max-symbols 5 --seed 7]
//   rnntg_cli decode --data DIR [--model neural:<seed>|lstm:<seed>]
//                    [--algo graph|label_loop_graph|tdt_label_loop_graph|
//                            sync_free|label_loop|tdt_label_loop|
//                            cpu:<any of the above>|cpu:baseline]
//                    [--exec tensor|persistent|graph|hostloop]
//                    [--hyp out.jsonl] [--report r.json] [--warmup 0] [--iters 1]
//                    [--max-symbols N] [--hidden-dim 32] [--embed-dim 16]
//                    [--joint-dim 32] [--layers 1] [--durations 0,1,2,3,4]
//   rnntg_cli compare a.jsonl b.jsonl      (prints "WER x"; exit 0 iff tokens
//                                           identical, 1 otherwise, 2 if the
//                                           utterance ids differ: cli.cpp:352-376)
//
// Datasets use the reference's own formats: manifest.json + TNSR tensor files
// (tensor.hpp:148-150), hypotheses JSONL via write/read_hypotheses_jsonl
// (decoders.cpp:770-811), WER via analysis.hpp:51.  GPU algorithms go through
// the C++ drop-in (include/rnntsim_cuda.hpp); the cpu: prefix runs the
// UNMODIFIED reference decoders on the same model for an end-to-end check.
// The CLI11 front end of the reference is not in this image, hence the small
// argv parser.  Models: neural:<seed> is the reference tanh NeuralModel
// (init_params, model.cpp:81-108); lstm:<seed> the LstmModel extension with
// weights from the oracle generator (same bytes on CPU and GPU).
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <map>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include <json.hpp>  // nlohmann/json 3.11.3, the copy the reference build uses

#include "cuda_lstm.hpp"
#include "rnnt_oracle.h"
#include "rnntsim/analysis.hpp"
#include "rnntsim/decoders.hpp"
#include "rnntsim/errors.hpp"
#include "rnntsim/model.hpp"
#include "rnntsim/tensor.hpp"
#include "rnntsim_cuda.hpp"

using namespace rnntsim;
using json = nlohmann::json;
namespace fs = std::filesystem;

namespace {

struct Args {
  std::string cmd;
  std::map<std::string, std::string> opt;
  std::vector<std::string> pos;
  std::string get(const std::string& k, const std::string& d) const {
    auto it = opt.find(k);
    return it == opt.end() ? d : it->second;
  }
  int geti(const std::string& k, int d) const { return std::stoi(get(k, std::to_string(d))); }
};

Args parse(int argc, char** argv) {
  Args a;
  if (argc < 2) throw ValueError("usage: rnntg_cli gen|decode|compare ...");
  a.cmd = argv[1];
  for (int i = 2; i < argc; ++i) {
    std::string s = argv[i];
    if (s.rfind("--", 0) == 0) {
      if (i + 1 >= argc) throw ValueError("missing value for " + s);
      a.opt[s.substr(2)] = argv[++i];
    } else {
      a.pos.push_back(s);
    }
  }
  return a;
}

std::vector<int> parse_int_list(const std::string& s) {
  std::vector<int> v;
  std::stringstream ss(s);
  std::string item;
  while (std::getline(ss, item, ','))
    if (!item.empty()) v.push_back(std::stoi(item));
  return v;
}

// -- gen (cli.cpp:95-170, random pattern) ------------------------------------
int cmd_gen(const Args& a) {
  const std::string out = a.get("out", "");
  if (out.empty()) throw ValueError("--out is required");
  const int batch = a.geti("batch", 8), frames = a.geti("frames", 32), fdim = a.geti("feature-dim", 16);
  const int vocab = a.geti("vocab", 16), ms = a.geti("max-symbols", 5);
  const uint64_t seed = std::stoull(a.get("seed", "7"));
  if (a.get("pattern", "random") != "random")
    throw ValueError("only the random pattern is generated (the adversarial one needs ScriptedModel)");
  fs::create_directories(out);
  json manifest;
  manifest["pattern"] = "random";
  manifest["vocab"] = vocab;
  manifest["max_symbols"] = ms;
  manifest["seed"] = seed;
  manifest["feature_dim"] = fdim;
  json records = json::array();
  Rng rng(seed);
  for (int b = 0; b < batch; ++b) {
    std::vector<float> data(static_cast<size_t>(frames) * fdim);
    for (float& v : data) v = rng.uniform(-1.0f, 1.0f);
    const int out_len = 1 + rng.uniform_int(frames);
    char name[32];
    std::snprintf(name, sizeof(name), "utt_%03d.tnsr", b);
    write_tensor_file(out + "/" + name, Tensor::from_floats(std::move(data), {frames, fdim}));
    json rec;
    std::snprintf(name, sizeof(name), "utt_%03d", b);
    rec["id"] = name;
    std::snprintf(name, sizeof(name), "utt_%03d.tnsr", b);
    rec["features"] = name;
    rec["out_len"] = out_len;
    records.push_back(rec);
  }
  manifest["records"] = records;
  std::ofstream os(out + "/manifest.json");
  if (!os) throw IoError("cannot write manifest in " + out);
  os << manifest.dump(2) << "\n";
  std::cout << "wrote " << records.size() << " utterances to " << out << "\n";
  return 0;
}

// -- dataset (cli.cpp:172-207) -------------------------------------------------
struct Dataset {
  std::vector<std::string> ids;
  Tensor x, out_len;
  int feature_dim = 0, vocab = 16, max_symbols = 5;
};

Dataset load_dataset(const std::string& dir) {
  std::ifstream is(dir + "/manifest.json");
  if (!is) throw IoError("cannot read " + dir + "/manifest.json");
  json m = json::parse(is, nullptr, false);
  if (m.is_discarded()) throw IoError("invalid manifest in " + dir);
  Dataset ds;
  ds.feature_dim = m.at("feature_dim").get<int>();
  ds.vocab = m.value("vocab", 16);
  ds.max_symbols = m.value("max_symbols", 5);
  std::vector<Tensor> feats;
  std::vector<int32_t> lens;
  for (const auto& rec : m.at("records")) {
    ds.ids.push_back(rec.at("id").get<std::string>());
    feats.push_back(read_tensor_file(dir + "/" + rec.at("features").get<std::string>()));
    lens.push_back(rec.at("out_len").get<int32_t>());
  }
  if (feats.empty()) throw ValueError("dataset has no records");
  const int64_t frames = feats[0].dim(0), width = feats[0].dim(1);
  for (const auto& f : feats)
    if (f.rank() != 2 || f.dim(0) != frames || f.dim(1) != width)
      throw DimensionError("all utterances must share [frames, feature_dim]");
  const int64_t batch = static_cast<int64_t>(feats.size());
  Tensor x(Dtype::Float32, {batch, frames, width});
  auto px = x.f32();
  for (int64_t b = 0; b < batch; ++b)
    std::copy_n(feats[static_cast<size_t>(b)].f32().data(), frames * width, &px[b * frames * width]);
  ds.x = std::move(x);
  ds.out_len = Tensor::from_ints(std::move(lens), {batch});
  return ds;
}

// -- models (cli.cpp:211-247 + the LSTM extension) ----------------------------
std::unique_ptr<DecoderModel> build_model(const Args& a, const Dataset& ds, bool tdt) {
  const std::string spec = a.get("model", "neural:1");
  const auto colon = spec.find(':');
  const std::string kind = spec.substr(0, colon);
  const uint64_t seed = colon == std::string::npos ? 1 : std::stoull(spec.substr(colon + 1));
  const std::vector<int> durs = tdt ? parse_int_list(a.get("durations", "0,1,2,3,4")) : std::vector<int>{};
  if (kind == "neural") {
    RnntDims dims;
    dims.vocab = ds.vocab;
    dims.embed = a.geti("embed-dim", 16);
    dims.hidden = a.geti("hidden-dim", 32);
    dims.joint = a.geti("joint-dim", 32);
    dims.feature = ds.feature_dim;
    dims.durations = durs;
    return std::make_unique<NeuralModel>(init_params(seed, dims));
  }
  if (kind == "lstm") {
    orc_dims d{};
    d.vocab = ds.vocab;
    d.embed = a.geti("embed-dim", 16);
    d.hidden = a.geti("hidden-dim", 32);
    d.joint = a.geti("joint-dim", 32);
    d.feature = ds.feature_dim;
    d.cell = 1;
    d.layers = a.geti("layers", 1);
    d.num_durations = static_cast<int>(durs.size());
    for (size_t i = 0; i < durs.size(); ++i) d.durations[i] = durs[i];
    if (orc_validate_dims(&d) != 0) throw ValueError("invalid LSTM dimensions");
    std::vector<std::vector<float>> w(orc_num_params(&d));
    std::vector<float*> ptr;
    for (int i = 0; i < (int)w.size(); ++i) {
      int64_t r = 0, c = 0;
      orc_param_size(&d, i, &r, &c);
      w[i].assign(static_cast<size_t>(r * c), 0.0f);
      ptr.push_back(w[i].data());
    }
    orc_init_params(seed, &d, ptr.data());
    return std::make_unique<CudaLstm>(d, std::move(w));
  }
  throw ValueError("model must be neural:<seed> or lstm:<seed>");
}

rnntg_exec parse_exec(const std::string& s) {
  if (s == "tensor") return RNNTG_EXEC_TENSOR;
  if (s == "persistent") return RNNTG_EXEC_PERSISTENT;
  if (s == "graph") return RNNTG_EXEC_GRAPH;
  if (s == "hostloop") return RNNTG_EXEC_HOSTLOOP;
  if (s == "graph-ffma") return RNNTG_EXEC_GRAPH_FFMA;
  throw ValueError("exec must be tensor, persistent, graph or hostloop");
}

// -- decode (cli.cpp:277-348) -------------------------------------------------
int cmd_decode(const Args& a) {
  const std::string data = a.get("data", "");
  if (data.empty()) throw ValueError("--data is required");
  std::string algo = a.get("algo", "graph");
  const int warmup = a.geti("warmup", 0), iters = a.geti("iters", 1);
  if (warmup < 0 || iters < 1) throw ValueError("warmup must be >= 0 and iters >= 1");
  const bool cpu = algo.rfind("cpu:", 0) == 0;
  if (cpu) algo = algo.substr(4);
  Dataset ds = load_dataset(data);
  const int ms = a.geti("max-symbols", 0) > 0 ? a.geti("max-symbols", 0) : ds.max_symbols;
  const bool tdt = algo.rfind("tdt", 0) == 0;
  auto model = build_model(a, ds, tdt);
  if (!cpu) cuda::set_executor(parse_exec(a.get("exec", "tensor")));
  static const std::map<std::string, DecodeAlgo> kGraph = {{"graph", DecodeAlgo::FrameSync},
                                                           {"label_loop_graph", DecodeAlgo::LabelLoop},
                                                           {"tdt_label_loop_graph", DecodeAlgo::TdtLabelLoop}};
  Engine engine;
  const int batch = static_cast<int>(ds.x.dim(0)), frames = static_cast<int>(ds.x.dim(1));
  Hypotheses hyps;
  std::vector<double> ms_runs;
  auto it = kGraph.find(algo);
  std::unique_ptr<CapturedDecoder> cap;
  if (it != kGraph.end())
    cap = std::make_unique<CapturedDecoder>(cpu ? build_decode_graph(engine, *model, it->second, batch, frames, ms)
                                                : cuda::build_decode_graph(engine, *model, it->second, batch,
                                                                           frames, ms));
  for (int i = 0; i < warmup + iters; ++i) {
    const auto t0 = std::chrono::steady_clock::now();
    if (cap) {
      hyps = cpu ? replay_decode(*cap, ds.x, ds.out_len) : cuda::replay_decode(*cap, ds.x, ds.out_len);
    } else if (algo == "sync_free") {
      hyps = cpu ? greedy_decode_sync_free(engine, *model, ds.x, ds.out_len, ms)
                 : cuda::greedy_decode_sync_free(engine, *model, ds.x, ds.out_len, ms);
    } else if (algo == "label_loop") {
      hyps = cpu ? label_looping_decode(engine, *model, ds.x, ds.out_len, ms)
                 : cuda::label_looping_decode(engine, *model, ds.x, ds.out_len, ms);
    } else if (algo == "tdt_label_loop") {
      hyps = cpu ? tdt_label_looping_decode(engine, *model, ds.x, ds.out_len, ms)
                 : cuda::tdt_label_looping_decode(engine, *model, ds.x, ds.out_len, ms);
    } else if (algo == "baseline" && cpu) {
      hyps = greedy_decode_baseline(engine, *model, ds.x, ds.out_len, ms);
    } else {
      throw ValueError("unknown algorithm: " + algo);
    }
    const auto t1 = std::chrono::steady_clock::now();
    if (i >= warmup) ms_runs.push_back(std::chrono::duration<double, std::milli>(t1 - t0).count());
  }
  const std::string hyp_path = a.get("hyp", "");
  if (!hyp_path.empty()) write_hypotheses_jsonl(hyp_path, ds.ids, hyps);
  double mean = 0.0;
  for (double v : ms_runs) mean += v / ms_runs.size();
  int64_t frames_total = 0;
  for (int32_t l : ds.out_len.i32()) frames_total += l;
  json report;
  report["algo"] = (cpu ? "cpu:" : "") + algo;
  report["exec"] = cpu ? "reference-cpu" : a.get("exec", "tensor");
  report["model"] = a.get("model", "neural:1");
  report["batch"] = batch;
  report["frames"] = frames;
  report["max_symbols"] = ms;
  report["warmup"] = warmup;
  report["iters"] = iters;
  report["wall_ms_mean"] = mean;  // host wall clock around each decode call (H2D + launch + D2H)
  report["frames_per_s"] = mean > 0 ? frames_total / (mean / 1000.0) : 0.0;
  if (!cpu) report["joint_evals"] = cuda::decode_joint_evals(engine);
  const std::string rep_path = a.get("report", "");
  if (!rep_path.empty()) {
    std::ofstream os(rep_path);
    if (!os) throw IoError("cannot write " + rep_path);
    os << report.dump(2) << "\n";
  }
  std::cout << report.dump() << "\n";
  return 0;
}

// -- compare (cli.cpp:352-376) ------------------------------------------------
int cmd_compare(const Args& a) {
  if (a.pos.size() != 2) throw ValueError("compare needs two hypothesis files");
  auto ha = read_hypotheses_jsonl(a.pos[0]);
  auto hb = read_hypotheses_jsonl(a.pos[1]);
  std::map<std::string, const Hypothesis*> by_id;
  for (const auto& [id, h] : hb) by_id[id] = &h;
  if (ha.size() != hb.size() || ha.size() != by_id.size()) {
    std::cerr << "utterance id sets differ\n";
    return 2;
  }
  Hypotheses refs, hyps;
  bool identical = true;
  for (const auto& [id, h] : ha) {
    auto it = by_id.find(id);
    if (it == by_id.end()) {
      std::cerr << "utterance id sets differ\n";
      return 2;
    }
    refs.push_back(h);
    hyps.push_back(*it->second);
    identical = identical && h.tokens == it->second->tokens;
  }
  std::cout << "WER " << wer(refs, hyps) << "\n";
  return identical ? 0 : 1;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    const Args a = parse(argc, argv);
    if (a.cmd == "gen") return cmd_gen(a);
    if (a.cmd == "decode") return cmd_decode(a);
    if (a.cmd == "compare") return cmd_compare(a);
    throw ValueError("unknown command " + a.cmd);
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 3;
  }
}
