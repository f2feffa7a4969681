// oracle/shim_driver.cpp -- TEST INFRASTRUCTURE ONLY: exercises the
// reference-side binding (integration/tec_sm100_shim.*) on whole reference
// graphs. Built by `make -C oracle shim` against the unmodified reference
// library (oracle/_ref/libtec_ref.a) and libtec_sm100.so.
//
//   eval <graph.json> <feeds_dir> <out_dir> [f32|f32tc]
//        graph_from_json -> fuse_pass (R/src/graph_passes.cpp:196) ->
//        tec_sm100_shim::evaluate_graph: conv-rooted fused nodes run as ONE
//        tec_eval_fused_conv each, every other node on the reference's own
//        eval_graph_node. Outputs saved like the reference's (save_tensor);
//        prints {"sm100_nodes": n, "nodes": total}.
//   check <graph.json> <feeds_dir> [f32|f32tc]
//        node-by-node parity on real graph data: walks the fused graph with
//        the REFERENCE's eval_graph_node and, for every conv-rooted fused
//        node, also runs the shim on the same (reference) inputs and
//        compares -- f32 bit-for-bit, f32tc with DenseTensor::same_values
//        (1e-4). Prints {"checked", "failed", "max_rel"}.
//   op <x_dir> <w_dir> <out_dir> <stride> <pad> [depthwise]
//        native_conv (the OperatorDef::native_eval hook) on x / w.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>

#include "tec/graph.hpp"
#include "tec/graph_passes.hpp"
#include "tec/io.hpp"
#include "tec_sm100_shim.hpp"

using namespace tec;

int main(int argc, char** argv) {
  try {
    std::string cmd = argc > 1 ? argv[1] : "";
    if (cmd == "eval" && (argc == 5 || argc == 6)) {
      ComputeGraph g = graph_from_json(parse_json(read_text_file(argv[2]), argv[2]));
      ComputeGraph f = fuse_pass(g);
      std::map<std::string, DenseTensor> feeds;
      for (const auto& n : f.nodes)
        if (n.op == "input") feeds.emplace(n.id, load_tensor(argv[3], n.id));
      tec_sm100_shim::Options opt;
      int64_t count = 0;
      opt.sm100_nodes = &count;
      if (argc == 6 && std::string(argv[5]) == "f32tc") opt.f32_compute = TEC_COMPUTE_F32TC;
      auto outs = tec_sm100_shim::evaluate_graph(f, feeds, opt);
      for (const auto& [id, t] : outs) save_tensor(argv[4], id, t);
      std::printf("{\"sm100_nodes\": %lld, \"nodes\": %zu}\n", (long long)count, f.nodes.size());
      return 0;
    }
    if (cmd == "check" && (argc == 4 || argc == 5)) {
      ComputeGraph f = fuse_pass(graph_from_json(parse_json(read_text_file(argv[2]), argv[2])));
      tec_sm100_shim::Options opt;
      const bool tc = argc == 5 && std::string(argv[4]) == "f32tc";
      if (tc) opt.f32_compute = TEC_COMPUTE_F32TC;
      std::map<std::string, DenseTensor> env;
      int checked = 0, failed = 0;
      double max_rel = 0.0;
      for (const auto& n : f.nodes) {
        if (n.op == "input") { env.emplace(n.id, load_tensor(argv[3], n.id)); continue; }
        if (n.op == "const") { env.emplace(n.id, *n.data); continue; }
        std::vector<DenseTensor> ins;
        for (const auto& in : n.inputs) ins.push_back(env.at(in));
        DenseTensor ref = tec::eval_graph_node(n, ins);
        if (tec_sm100_shim::is_sm100_fused(n)) {
          DenseTensor got = tec_sm100_shim::eval_graph_node(n, ins, opt);
          ++checked;
          bool ok;
          if (!tc || !got.is_float()) {
            ok = got.is_float() ? std::memcmp(got.f_data().data(), ref.f_data().data(),
                                              ref.f_data().size() * 4) == 0
                                : got.i_data() == ref.i_data();
          } else {
            ok = got.same_values(ref, 1e-4);
            for (size_t i = 0; i < ref.f_data().size(); ++i) {
              const double a = got.f_data()[i], b = ref.f_data()[i];
              max_rel = std::max(max_rel, std::fabs(a - b) /
                                              std::max({std::fabs(a), std::fabs(b), 1.0}));
            }
          }
          failed += !ok;
        }
        env.insert_or_assign(n.id, std::move(ref));
      }
      std::printf("{\"checked\": %d, \"failed\": %d, \"max_rel\": %.6g}\n", checked, failed,
                  max_rel);
      return 0;
    }
    if (cmd == "op" && (argc == 7 || argc == 8)) {
      DenseTensor x = load_tensor(argv[2], "x"), w = load_tensor(argv[3], "w");
      AttrMap a;
      a["strides"] = std::vector<int64_t>{std::stoll(argv[5]), std::stoll(argv[5])};
      a["padding"] = std::vector<int64_t>{std::stoll(argv[6]), std::stoll(argv[6])};
      DenseTensor y = tec_sm100_shim::native_conv({x, w}, a, argc == 8);
      save_tensor(argv[4], "y", y);
      return 0;
    }
    std::fprintf(stderr, "usage: shim_driver eval <graph> <feeds> <out> [f32|f32tc] | op ...\n");
    return 2;
  } catch (const Error& e) {
    std::fprintf(stderr, "tec::Error %d %s\n", static_cast<int>(e.code()), e.what());
    return 3;
  }
}
