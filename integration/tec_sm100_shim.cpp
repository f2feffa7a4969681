// tec_sm100_shim.cpp -- see tec_sm100_shim.hpp.
#include "tec_sm100_shim.hpp"

#include <string>

#include "tec/error.hpp"

namespace tec_sm100_shim {

void check(tec_status st) {
  if (st == TEC_OK) return;
  const char* msg = tec_last_error();
  if (st >= 1 && st <= (int)tec::ErrorCode::kInternal + 1)
    tec::fail(static_cast<tec::ErrorCode>(st - 1), std::string("sm100: ") + msg);
  tec::fail(tec::ErrorCode::kInternal, std::string("sm100 (CUDA): ") + msg);
}

namespace {

tec_conv_desc make_desc(const tec::DenseTensor& x, const tec::DenseTensor& w,
                        const tec::AttrMap& attrs, bool depthwise, const Options& opt) {
  auto st = tec::attr_ints(attrs, "strides", {1, 1});
  auto pd = tec::attr_ints(attrs, "padding", {0, 0});
  if (x.shape().size() != 4 || w.shape().size() != 4 || st.size() != 2 || pd.size() != 2)
    tec::fail(tec::ErrorCode::kShapeMismatch, "conv wants NCHW data, OIHW weights, pairs");
  if (x.dtype() != w.dtype())
    tec::fail(tec::ErrorCode::kShapeMismatch, "conv operand dtypes differ");
  tec_conv_desc d{};
  d.n = x.shape()[0]; d.c = x.shape()[1]; d.h = x.shape()[2]; d.w = x.shape()[3];
  d.k = w.shape()[0]; d.r = w.shape()[2]; d.s = w.shape()[3];
  d.stride_h = st[0]; d.stride_w = st[1]; d.pad_h = pd[0]; d.pad_w = pd[1];
  d.depthwise = depthwise ? 1 : 0;
  d.compute = x.dtype() == tec::DType::kI8 ? TEC_COMPUTE_I8 : opt.f32_compute;
  if (depthwise && w.shape()[1] != 1)
    tec::fail(tec::ErrorCode::kShapeMismatch, "depthwise_conv2d weights must be [C,1,kh,kw]");
  if (!depthwise && w.shape()[1] != x.shape()[1])
    tec::fail(tec::ErrorCode::kShapeMismatch, "conv2d: weight input-channel dim mismatch");
  return d;
}

// Host operand bytes in the layout tec_eval_fused_conv takes: f32 as is, i8
// packed to 1 byte/elem (the DenseTensor keeps int32 storage), i32 as is.
const void* host_ptr(const tec::DenseTensor& t, std::vector<uint8_t>* keep) {
  if (t.dtype() == tec::DType::kF32) return t.f_data().data();
  if (t.dtype() == tec::DType::kI8) {
    *keep = t.to_bytes();
    return keep->data();
  }
  return t.i_data().data();
}

tec::DenseTensor run_fused(const tec::DenseTensor& x, const tec::DenseTensor& w,
                           const tec::AttrMap& attrs, bool depthwise,
                           const tec_epilogue* epi, const Options& opt) {
  tec_conv_desc d = make_desc(x, w, attrs, depthwise, opt);
  int64_t os[4];
  check(tec_conv_infer(&d, os));
  const bool integer = x.dtype() == tec::DType::kI8;
  tec::DenseTensor y(tec::TensorType({os[0], os[1], os[2], os[3]},
                                     integer ? tec::DType::kI32 : tec::DType::kF32));
  std::vector<uint8_t> xb, wb;
  void* yp = integer ? (void*)y.i_data().data() : (void*)y.f_data().data();
  check(tec_eval_fused_conv(&d, epi, nullptr, host_ptr(x, &xb), host_ptr(w, &wb), yp,
                            opt.device));
  if (opt.sm100_nodes) ++*opt.sm100_nodes;
  return y;
}

int epi_code(const std::string& op) {
  if (op == "scale") return TEC_EPI_SCALE;
  if (op == "bias_add") return TEC_EPI_BIAS;
  if (op == "add") return TEC_EPI_ADD;
  if (op == "mul") return TEC_EPI_MUL;
  if (op == "relu") return TEC_EPI_RELU;
  return 0;
}

}  // namespace

tec::DenseTensor native_conv(const std::vector<tec::DenseTensor>& inputs,
                             const tec::AttrMap& attrs, bool depthwise, const Options& opt) {
  if (inputs.size() != 2)
    tec::fail(tec::ErrorCode::kShapeMismatch, "conv expects 2 inputs");
  return run_fused(inputs[0], inputs[1], attrs, depthwise, nullptr, opt);
}

bool is_sm100_fused(const tec::GraphNode& n) {
  if (n.op != "fused" || n.members.empty()) return false;
  const auto& root = n.members[0].op;
  if (root != "conv2d" && root != "depthwise_conv2d") return false;
  if (n.members.size() > (size_t)TEC_MAX_EPILOGUE + 1) return false;
  int counts[6] = {0, 0, 0, 0, 0, 0};
  std::string prev = n.members[0].id;
  for (size_t i = 1; i < n.members.size(); ++i) {
    const auto& m = n.members[i];
    const int code = epi_code(m.op);
    if (!code) return false;
    // one operand slot per kind in tec_epilogue
    if (code != TEC_EPI_RELU && code != TEC_EPI_SCALE && ++counts[code] > 1) return false;
    bool chained = false;
    for (const auto& in : m.inputs) chained |= in == prev;
    if (!chained) return false;
    prev = m.id;
  }
  return true;
}

tec::DenseTensor eval_graph_node(const tec::GraphNode& n,
                                 const std::vector<tec::DenseTensor>& inputs,
                                 const Options& opt) {
  if (!is_sm100_fused(n)) return tec::eval_graph_node(n, inputs);  // reference path
  std::map<std::string, const tec::DenseTensor*> env;
  for (size_t i = 0; i < n.inputs.size(); ++i) env[n.inputs[i]] = &inputs[i];
  const tec::GraphNode& root = n.members[0];
  tec_epilogue e{};
  std::string prev = root.id;
  for (size_t i = 1; i < n.members.size(); ++i) {
    const tec::GraphNode& m = n.members[i];
    const int code = epi_code(m.op);
    e.ops[e.n_ops] = code;
    if (code == TEC_EPI_SCALE) e.scale[e.n_ops] = tec::attr_double(m.attrs, "scale", 1.0);
    for (const auto& in : m.inputs) {
      if (in == prev) continue;
      auto it = env.find(in);
      if (it == env.end())
        tec::fail(tec::ErrorCode::kLoweringError, "member reads an internal tensor");
      const tec::DenseTensor& t = *it->second;
      const void* p = t.is_float() ? (const void*)t.f_data().data() : (const void*)t.i_data().data();
      if (code == TEC_EPI_BIAS) e.bias = p;
      else if (code == TEC_EPI_ADD) e.residual = p;
      else if (code == TEC_EPI_MUL) e.mul_operand = p;
    }
    ++e.n_ops;
    prev = m.id;
  }
  return run_fused(*env.at(root.inputs[0]), *env.at(root.inputs[1]), root.attrs,
                   root.op == "depthwise_conv2d", &e, opt);
}

std::map<std::string, tec::DenseTensor> evaluate_graph(
    const tec::ComputeGraph& g, const std::map<std::string, tec::DenseTensor>& feeds,
    const Options& opt) {
  std::map<std::string, tec::DenseTensor> env;
  for (const auto& n : g.nodes) {
    if (n.op == "input") {
      auto it = feeds.find(n.id);
      if (it == feeds.end())
        tec::fail(tec::ErrorCode::kIOError, "no value for graph input '" + n.id + "'");
      if (it->second.type() != n.out_type)
        tec::fail(tec::ErrorCode::kShapeMismatch, "input " + n.id + " has the wrong type");
      env.emplace(n.id, it->second);
      continue;
    }
    if (n.op == "const") {
      if (!n.data)
        tec::fail(tec::ErrorCode::kNotEnoughData, "const node '" + n.id + "' carries no data");
      env.emplace(n.id, *n.data);
      continue;
    }
    std::vector<tec::DenseTensor> ins;
    for (const auto& in : n.inputs) ins.push_back(env.at(in));
    env.insert_or_assign(n.id, eval_graph_node(n, ins, opt));
  }
  std::map<std::string, tec::DenseTensor> out;
  for (const auto& o : g.outputs) out.emplace(o, env.at(o));
  return out;
}

}  // namespace tec_sm100_shim
