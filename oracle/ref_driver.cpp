// oracle/ref_driver.cpp -- TEST INFRASTRUCTURE ONLY (never shipped, never on
// the product path).
//
// A small command-line front end over the UNMODIFIED reference library
// (tec, /root/reference/proj/src/*.cpp, compiled in place by oracle/Makefile
// into oracle/_ref/). It exists so the test-suite and bench.py's reference
// arm can run the reference's own CPU path:
//
//   eval  <graph.json> <feeds_dir> <out_dir>
//         graph_from_json (R/src/graph.cpp:189) -> evaluate_graph
//         (R/src/graph.cpp:227); every graph input `id` is read with
//         load_tensor(feeds_dir, id) (R/src/io.cpp:121) and every output is
//         written with save_tensor (R/src/io.cpp:111).
//   fuse  <graph.json> <out.json>
//         fuse_pass (R/src/graph_passes.cpp:196) + plan_memory (:285); writes
//         {"graph": graph_to_json(fused), "plan": {...}}.
//   fold  <graph.json> <out.json>
//         fold_constants (R/src/graph_passes.cpp:41-73); writes graph_to_json.
//   layouts <graph.json> <prefs.json> <out.json>
//         apply_layouts (R/src/graph_passes.cpp:84-178) with {node: layout}.
//   gen   <out_dir> <name> <dtype> <seed> <d0> [d1 ...]
//         random_tensor (R/src/tensor.cpp:74) with mt19937_64(seed), saved
//         with save_tensor -- the reference's own synthetic distributions.
//   gbt   <in.json> <out.json>
//         CostModel::train / predict / pairwise_rank_accuracy
//         (R/src/gbt.cpp:119-246) on {"feats", "costs", "query", "params"};
//         writes {"pred", "acc", "model"} -- pins the tuner's restatement.
//   sched <in.json> <out_dir>
//         a B200 Config's schedule log (tuner.schedule_log) replayed on the
//         reference: conv2d compute "conv" over placeholders D / W
//         (make_conv), Schedule::replay (R/src/schedule.cpp:486-491) ->
//         lower(target "interp") -> interpret (R/src/interp.cpp:501-546) on
//         random_tensor feeds; saves D, W, interp and reference outputs;
//         prints {"features": extract_features, "log", "cost", "matches"} --
//         the legality check, the reference features and the second oracle.
//   serve <seconds>
//         the reference's own WorkerServer (R/src/rpc.cpp:129-181) on an
//         ephemeral 127.0.0.1 port, printed as {"port": p}; stops after
//         <seconds> -- pins the RPC framing of paper_1802_04799_b200/rpc.py.
//   bench <op> <C> <H> <W> <OC> <K> <stride> <pad> <rows> <seed> [dtype]
//         times eval_graph_node (R/src/graph.cpp:209) on the fused node
//         [conv2d|depthwise_conv2d, bias_add, relu] built exactly as
//         fuse_pass emits it, on a bounded sample: batch 1, full width and
//         channels, `rows` output rows. Prints one JSON line.
#include <chrono>
#include <cstdio>
#include <iostream>
#include <random>
#include <string>
#include <vector>

#include "tec/autotune.hpp"
#include "tec/graph.hpp"
#include "tec/interp.hpp"
#include "tec/lower.hpp"
#include "tec/rpc.hpp"
#include "tec/schedule.hpp"
#include <thread>
#include "tec/texpr.hpp"
#include "tec/graph_passes.hpp"
#include "tec/io.hpp"
#include "tec/ops.hpp"
#include "tec/tensor.hpp"

using namespace tec;

static int cmd_eval(const std::string& gpath, const std::string& feeds_dir,
                    const std::string& out_dir) {
  ComputeGraph g = graph_from_json(parse_json(read_text_file(gpath), gpath));
  std::map<std::string, DenseTensor> feeds;
  for (const auto& n : g.nodes)
    if (n.op == "input") feeds.emplace(n.id, load_tensor(feeds_dir, n.id));
  auto outs = evaluate_graph(g, feeds);
  for (const auto& [id, t] : outs) save_tensor(out_dir, id, t);
  return 0;
}

static int cmd_fuse(const std::string& gpath, const std::string& out_path) {
  ComputeGraph g = graph_from_json(parse_json(read_text_file(gpath), gpath));
  ComputeGraph f = fuse_pass(g);
  MemoryPlan p = plan_memory(f);
  check_memory_plan(f, p);
  nlohmann::json j;
  j["graph"] = graph_to_json(f);
  j["plan"] = {{"slot_of", p.slot_of},
               {"slot_bytes", p.slot_bytes},
               {"total_bytes", p.total_bytes},
               {"naive_bytes", p.naive_bytes}};
  write_text_file(out_path, j.dump(1) + "\n");
  return 0;
}

static int cmd_fold(const std::string& gpath, const std::string& out_path) {
  ComputeGraph g = graph_from_json(parse_json(read_text_file(gpath), gpath));
  write_text_file(out_path, graph_to_json(fold_constants(g)).dump(1) + "\n");
  return 0;
}

static int cmd_layouts(const std::string& gpath, const std::string& ppath,
                       const std::string& out_path) {
  ComputeGraph g = graph_from_json(parse_json(read_text_file(gpath), gpath));
  nlohmann::json pj = parse_json(read_text_file(ppath), ppath);
  std::map<std::string, std::string> prefs;
  for (auto it = pj.begin(); it != pj.end(); ++it) prefs[it.key()] = it.value().get<std::string>();
  write_text_file(out_path, graph_to_json(apply_layouts(g, prefs)).dump(1) + "\n");
  return 0;
}

static int cmd_gbt(const std::string& in_path, const std::string& out_path) {
  nlohmann::json j = parse_json(read_text_file(in_path), in_path);
  GbtParams prm;
  if (j.contains("params")) {
    const auto& p = j["params"];
    prm.max_depth = p.value("max_depth", prm.max_depth);
    prm.rounds = p.value("rounds", prm.rounds);
    prm.learning_rate = p.value("learning_rate", prm.learning_rate);
    prm.reg_lambda = p.value("reg_lambda", prm.reg_lambda);
  }
  std::vector<FeatureVector> feats;
  for (const auto& r : j.at("feats")) feats.push_back(r.get<std::vector<double>>());
  std::vector<double> costs = j.at("costs").get<std::vector<double>>();
  CostModel m(prm);
  m.train(feats, costs);
  nlohmann::json out;
  std::vector<double> pred;
  for (const auto& r : j.at("query")) pred.push_back(m.predict(r.get<std::vector<double>>()));
  out["pred"] = pred;
  out["acc"] = pairwise_rank_accuracy(m, feats, costs);
  out["model"] = m.to_json();
  write_text_file(out_path, out.dump(1) + "\n");
  return 0;
}

static int cmd_sched(const std::string& in_path, const std::string& out_dir) {
  nlohmann::json j = parse_json(read_text_file(in_path), in_path);
  auto xs = j.at("x_shape").get<std::vector<int64_t>>();
  auto ws = j.at("w_shape").get<std::vector<int64_t>>();
  Tensor d = placeholder("D", TensorType(xs, DType::kF32));
  Tensor w = placeholder("W", TensorType(ws, DType::kF32));
  AttrMap a;
  a["strides"] = j.at("strides").get<std::vector<int64_t>>();
  a["padding"] = j.at("padding").get<std::vector<int64_t>>();
  Tensor conv = op_def("conv2d").make_compute("conv", {d, w}, a);
  Schedule s = Schedule::replay({conv}, j.at("log"));
  LoopProgram prog = lower(s, "conv");
  std::mt19937_64 rng(j.value("seed", 0));
  std::map<std::string, DenseTensor> feeds;
  feeds.emplace("D", random_tensor(d->type, rng));
  feeds.emplace("W", random_tensor(w->type, rng));
  InterpResult r = interpret(prog, feeds);
  DenseTensor want = evaluate_reference(conv, feeds);
  const DenseTensor& got = r.outputs.at("conv");
  save_tensor(out_dir, "D", feeds.at("D"));
  save_tensor(out_dir, "W", feeds.at("W"));
  save_tensor(out_dir, "interp", got);
  save_tensor(out_dir, "ref", want);
  nlohmann::json out;
  out["features"] = extract_features(prog);
  out["log"] = s.log();
  out["cost"] = r.cost();
  out["matches_1e5"] = got.same_values(want, 1e-5);
  std::printf("%s\n", out.dump().c_str());
  return 0;
}

static int cmd_serve(int seconds) {
  WorkerServer srv(0);
  std::printf("{\"port\": %d}\n", srv.port());
  std::fflush(stdout);
  std::this_thread::sleep_for(std::chrono::seconds(seconds));
  srv.stop();
  return 0;
}

static int cmd_gen(int argc, char** argv) {
  std::string dir = argv[2], name = argv[3];
  DType dt = dtype_from_name(argv[4]);
  uint64_t seed = std::stoull(argv[5]);
  std::vector<int64_t> shape;
  for (int i = 6; i < argc; ++i) shape.push_back(std::stoll(argv[i]));
  std::mt19937_64 rng(seed);
  save_tensor(dir, name, random_tensor(TensorType(shape, dt), rng));
  return 0;
}

static int cmd_bench(int argc, char** argv) {
  std::string op = argv[2];
  const int64_t C = std::stoll(argv[3]), H = std::stoll(argv[4]),
                W = std::stoll(argv[5]), OC = std::stoll(argv[6]),
                K = std::stoll(argv[7]), S = std::stoll(argv[8]),
                P = std::stoll(argv[9]), rows = std::stoll(argv[10]);
  const uint64_t seed = std::stoull(argv[11]);
  DType dt = argc > 12 ? dtype_from_name(argv[12]) : DType::kF32;
  const bool dw = op == "depthwise_conv2d";
  // Bounded sample: input rows so that exactly `rows` output rows exist.
  int64_t Hs = (rows - 1) * S + K - 2 * P;
  if (Hs < 1) Hs = 1;
  if (Hs > H) Hs = H;
  std::mt19937_64 rng(seed);
  DenseTensor x = random_tensor(TensorType({1, C, Hs, W}, dt), rng);
  DenseTensor w = random_tensor(
      TensorType({dw ? C : OC, dw ? 1 : C, K, K}, dt), rng);
  DType acc = dt == DType::kI8 ? DType::kI32 : dt;
  DenseTensor b = random_tensor(TensorType({dw ? C : OC}, acc), rng);

  GraphNode conv{.id = "conv", .op = op, .inputs = {"x", "w"}};
  conv.attrs["strides"] = std::vector<int64_t>{S, S};
  conv.attrs["padding"] = std::vector<int64_t>{P, P};
  GraphNode bias{.id = "bias", .op = "bias_add", .inputs = {"conv", "b"}};
  GraphNode relu{.id = "relu", .op = "relu", .inputs = {"bias"}};
  GraphNode fused{.id = "relu", .op = "fused", .inputs = {"x", "w", "b"}};
  fused.members = {conv, bias, relu};

  auto t0 = std::chrono::steady_clock::now();
  DenseTensor y = eval_graph_node(fused, {x, w, b});
  auto t1 = std::chrono::steady_clock::now();
  const double sec = std::chrono::duration<double>(t1 - t0).count();
  const auto& ys = y.shape();
  const int64_t outs = ys[0] * ys[1] * ys[2] * ys[3];
  const int64_t macs = outs * (dw ? 1 : C) * K * K;
  double checksum = 0;
  for (int64_t i = 0; i < outs; ++i) checksum += y.scalar_at(i);
  std::printf(
      "{\"op\": \"%s\", \"out_shape\": [%lld, %lld, %lld, %lld], "
      "\"macs\": %lld, \"seconds\": %.6f, \"checksum\": %.6f}\n",
      op.c_str(), (long long)ys[0], (long long)ys[1], (long long)ys[2],
      (long long)ys[3], (long long)macs, sec, checksum);
  return 0;
}

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: ref_driver eval|fuse|gen|bench ...\n");
    return 2;
  }
  try {
    std::string cmd = argv[1];
    if (cmd == "eval" && argc == 5) return cmd_eval(argv[2], argv[3], argv[4]);
    if (cmd == "fuse" && argc == 4) return cmd_fuse(argv[2], argv[3]);
    if (cmd == "fold" && argc == 4) return cmd_fold(argv[2], argv[3]);
    if (cmd == "layouts" && argc == 5) return cmd_layouts(argv[2], argv[3], argv[4]);
    if (cmd == "gen" && argc >= 7) return cmd_gen(argc, argv);
    if (cmd == "gbt" && argc == 4) return cmd_gbt(argv[2], argv[3]);
    if (cmd == "sched" && argc == 4) return cmd_sched(argv[2], argv[3]);
    if (cmd == "serve" && argc == 3) return cmd_serve(std::stoi(argv[2]));
    if (cmd == "bench" && argc >= 12) return cmd_bench(argc, argv);
    std::fprintf(stderr, "bad arguments for '%s'\n", cmd.c_str());
    return 2;
  } catch (const Error& e) {
    // Mirror the reference's error taxonomy on stderr for the tests.
    std::fprintf(stderr, "tec::Error %d %s\n", static_cast<int>(e.code()),
                 e.what());
    return 3;
  }
}
