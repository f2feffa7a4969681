// tec_sm100_shim.hpp -- the reference-side binding of the sm100 backend: the
// C++ a tec maintainer adds to route the fused-conv path through
// include/tec_sm100.h. It is compiled against the
// reference's own headers (/root/reference/proj/include) and linked against
// the unmodified reference library plus libtec_sm100.so; oracle/Makefile
// (`shim`) builds it with a small driver so the test-suite can run whole
// reference graphs through it (tests/test_integration_gpu.py).
//
//   native_conv       the OperatorDef::native_eval hook for conv2d /
//                     depthwise_conv2d (R/include/tec/ops.hpp:63-67,
//                     short-circuited by eval_operator, R/src/ops.cpp:520-521)
//   eval_graph_node   eval_graph_node for target sm100 (R/src/graph.cpp:209-225):
//                     a conv-rooted fused node is ONE tec_eval_fused_conv call,
//                     every other node the reference's own eval_graph_node
//   evaluate_graph    evaluate_graph (R/src/graph.cpp:227-256), same walk
#pragma once

#include <cstdint>
#include <map>
#include <string>
#include <vector>

#include "tec/graph.hpp"
#include "tec/ops.hpp"
#include "tec/tensor.hpp"
#include "tec_sm100.h"

namespace tec_sm100_shim {

struct Options {
  int device = 0;
  // f32 graphs: TEC_COMPUTE_F32 (bit-identical to evaluate_reference) or
  // TEC_COMPUTE_F32TC (tensor cores, 1e-4); i8 always runs TEC_COMPUTE_I8.
  int32_t f32_compute = TEC_COMPUTE_F32;
  int64_t* sm100_nodes = nullptr;  // optional count of nodes run on the GPU
};

// tec_status -> tec::Error with the same ErrorCode (1 + code, tec_sm100.h).
void check(tec_status st);

tec::DenseTensor native_conv(const std::vector<tec::DenseTensor>& inputs,
                             const tec::AttrMap& attrs, bool depthwise,
                             const Options& opt = Options());

// true when `n` is a fused node the sm100 path runs in one call
bool is_sm100_fused(const tec::GraphNode& n);

tec::DenseTensor eval_graph_node(const tec::GraphNode& n,
                                 const std::vector<tec::DenseTensor>& inputs,
                                 const Options& opt = Options());

std::map<std::string, tec::DenseTensor> evaluate_graph(
    const tec::ComputeGraph& g, const std::map<std::string, tec::DenseTensor>& feeds,
    const Options& opt = Options());

}  // namespace tec_sm100_shim
