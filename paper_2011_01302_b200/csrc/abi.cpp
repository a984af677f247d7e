// extern "C" entry points of include/ios.h. No exception crosses this boundary.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <sstream>

#include "ios_core.h"

namespace ios {
int pool_out_size(int h, int k, int s, int p, bool ceil_mode);
const char* last_error_cstr();
}  // namespace ios

using namespace ios;

struct ios_graph_s {
  Graph g;
};
struct ios_schedule_s {
  Schedule q;
};

#define ABI_BEGIN try {
#define ABI_END                                \
  }                                            \
  catch (const ios::Error& e) {                \
    set_error(e.msg);                          \
    return e.code;                             \
  }                                            \
  catch (const std::bad_alloc&) {              \
    set_error("host out of memory");           \
    return IOS_ERR_OOM;                        \
  }                                            \
  catch (const std::exception& e) {            \
    set_error(e.what());                       \
    return IOS_ERR_INVALID_ARG;                \
  }                                            \
  return IOS_OK;

#define REQUIRE(cond, msg) \
  if (!(cond)) IOS_FAIL(IOS_ERR_INVALID_ARG, msg)

namespace {

// Shape inference for one op (Sec. 3 semantics; conv/pool output sizes as DESIGN.md Z11).
void infer_shape(Graph& g, Op& o) {
  const Op& x = g.ops[o.inputs[0]];
  o.N = x.N;
  switch (o.kind) {
    case IOS_OP_CONV: {
      REQUIRE(o.cout > 0 && o.kh > 0 && o.kw > 0 && o.sh > 0 && o.sw > 0 && o.ph >= 0 && o.pw >= 0, "bad conv parameters");
      if (o.inputs.size() != 1) IOS_FAIL(IOS_ERR_SHAPE, "conv takes one input");
      o.C = o.cout;
      o.H = (x.H + 2 * o.ph - o.kh) / o.sh + 1;
      o.W = (x.W + 2 * o.pw - o.kw) / o.sw + 1;
      if ((long)o.weight.size() != (long)o.cout * x.C * o.kh * o.kw) IOS_FAIL(IOS_ERR_SHAPE, "conv weight size mismatch");
      break;
    }
    case IOS_OP_SEPCONV: {
      REQUIRE(o.cout > 0 && o.kh > 0 && o.kw > 0 && o.sh > 0 && o.sw > 0, "bad sepconv parameters");
      for (int u : o.inputs) {
        const Op& y = g.ops[u];
        if (y.C != x.C || y.H != x.H || y.W != x.W) IOS_FAIL(IOS_ERR_SHAPE, "sepconv inputs differ in shape");
      }
      o.C = o.cout;
      o.H = (x.H + 2 * o.ph - o.kh) / o.sh + 1;
      o.W = (x.W + 2 * o.pw - o.kw) / o.sw + 1;
      if ((long)o.weight.size() != (long)x.C * o.kh * o.kw + (long)o.cout * x.C) IOS_FAIL(IOS_ERR_SHAPE, "sepconv weight size mismatch");
      break;
    }
    case IOS_OP_MAXPOOL:
    case IOS_OP_AVGPOOL: {
      REQUIRE(o.kh > 0 && o.kw > 0 && o.sh > 0 && o.sw > 0, "bad pool parameters");
      if (o.inputs.size() != 1) IOS_FAIL(IOS_ERR_SHAPE, "pool takes one input");
      const bool ceil = (o.flags & IOS_F_CEIL_MODE) != 0;
      o.C = x.C;
      o.H = pool_out_size(x.H, o.kh, o.sh, o.ph, ceil);
      o.W = pool_out_size(x.W, o.kw, o.sw, o.pw, ceil);
      break;
    }
    case IOS_OP_GLOBAL_AVGPOOL:
      if (o.inputs.size() != 1) IOS_FAIL(IOS_ERR_SHAPE, "global avgpool takes one input");
      o.C = x.C;
      o.H = o.W = 1;
      break;
    case IOS_OP_ADD:
    case IOS_OP_IDENTITY:
      for (int u : o.inputs) {
        const Op& y = g.ops[u];
        if (y.C != x.C || y.H != x.H || y.W != x.W) IOS_FAIL(IOS_ERR_SHAPE, "add inputs differ in shape");
      }
      if (o.kind == IOS_OP_IDENTITY && o.inputs.size() != 1) IOS_FAIL(IOS_ERR_SHAPE, "identity takes one input");
      o.C = x.C;
      o.H = x.H;
      o.W = x.W;
      break;
    case IOS_OP_CONCAT: {
      int c = 0;
      for (int u : o.inputs) {
        const Op& y = g.ops[u];
        if (y.H != x.H || y.W != x.W) IOS_FAIL(IOS_ERR_SHAPE, "concat inputs differ in H x W");
        c += y.C;
      }
      o.C = c;
      o.H = x.H;
      o.W = x.W;
      break;
    }
    case IOS_OP_LINEAR:
      if (o.inputs.size() != 1) IOS_FAIL(IOS_ERR_SHAPE, "linear takes one input");
      if (x.H != 1 || x.W != 1) IOS_FAIL(IOS_ERR_UNSUPPORTED, "linear needs a 1x1 spatial input (global pool first)");
      if ((long)o.weight.size() != (long)o.cout * x.C) IOS_FAIL(IOS_ERR_SHAPE, "linear weight size mismatch");
      o.C = o.cout;
      o.H = o.W = 1;
      o.kh = o.kw = o.sh = o.sw = 1;
      o.ph = o.pw = 0;
      break;
    default:
      IOS_FAIL(IOS_ERR_INVALID_ARG, "unknown op kind");
  }
  if (o.H < 1 || o.W < 1) IOS_FAIL(IOS_ERR_SHAPE, "empty output");
  if (o.kind == IOS_OP_ADD && !o.add_w.empty() && o.add_w.size() != o.inputs.size())
    IOS_FAIL(IOS_ERR_INVALID_ARG, "add_weights length");
  o.Cp = round_up(o.C, 8);
}

}  // namespace

extern "C" {

const char* ios_last_error(void) { return last_error_cstr(); }

ios_status ios_graph_create(int32_t batch, int32_t c, int32_t h, int32_t w, ios_math math, int32_t device,
                            ios_graph* out) {
  ABI_BEGIN
  REQUIRE(out && batch > 0 && c > 0 && h > 0 && w > 0, "bad graph input shape");
  REQUIRE(math == IOS_MATH_TF32 || math == IOS_MATH_BF16 || math == IOS_MATH_FP32_SIMT, "bad math mode");
  auto* gh = new ios_graph_s();
  Graph& g = gh->g;
  g.batch = batch;
  g.c = c;
  g.h = h;
  g.w = w;
  g.math = math;
  g.device = device;
  Op in;
  in.id = 0;
  in.kind = -1;
  in.block = -1;
  in.N = batch;
  in.C = c;
  in.H = h;
  in.W = w;
  in.Cp = round_up(c, 8);
  in.name = "input";
  g.ops.push_back(in);
  g.op_block_pos.push_back(-1);
  g.op_local.push_back(-1);
  *out = gh;
  ABI_END
}

ios_status ios_add_op(ios_graph gh, const ios_op_desc* d, const int32_t* inputs, int32_t n_inputs, int32_t* out_op_id) {
  ABI_BEGIN
  REQUIRE(gh && d && out_op_id && n_inputs >= 1 && inputs, "bad arguments");
  Graph& g = gh->g;
  Op o;
  o.id = (int)g.ops.size();
  o.kind = d->kind;
  o.block = d->block;
  o.cout = d->out_channels;
  o.kh = d->kernel_h;
  o.kw = d->kernel_w;
  o.sh = d->stride_h;
  o.sw = d->stride_w;
  o.ph = d->pad_h;
  o.pw = d->pad_w;
  o.flags = d->flags;
  if (o.kind == IOS_OP_SEPCONV) o.flags |= IOS_F_RELU_PRE;   // Relu-SepConv
  for (int i = 0; i < n_inputs; ++i) {
    if (inputs[i] < 0 || inputs[i] >= o.id) IOS_FAIL(IOS_ERR_DANGLING_INPUT, "input id " + std::to_string(inputs[i]) + " does not exist");
    o.inputs.push_back(inputs[i]);
  }
  if (o.kind < IOS_OP_CONV || o.kind > IOS_OP_LINEAR) IOS_FAIL(IOS_ERR_INVALID_ARG, "unknown op kind");
  const Op& x = g.ops[o.inputs[0]];
  long wsize = 0;
  if (o.kind == IOS_OP_CONV) wsize = (long)d->out_channels * x.C * d->kernel_h * d->kernel_w;
  if (o.kind == IOS_OP_SEPCONV) wsize = (long)x.C * d->kernel_h * d->kernel_w + (long)d->out_channels * x.C;
  if (o.kind == IOS_OP_LINEAR) wsize = (long)d->out_channels * x.C;
  if (wsize > 0) {
    REQUIRE(d->weight != nullptr, "weights required");
    o.weight.assign(d->weight, d->weight + wsize);
    o.bias.assign(d->out_channels, 0.0f);
    if (d->bias) o.bias.assign(d->bias, d->bias + d->out_channels);
  }
  if ((o.kind == IOS_OP_ADD || o.kind == IOS_OP_SEPCONV) && d->add_weights)
    o.add_w.assign(d->add_weights, d->add_weights + n_inputs);
  // blocks: contiguous in insertion order; edges only to the same or a later block
  auto it = g.block_pos.find(o.block);
  int bpos;
  if (it == g.block_pos.end()) {
    bpos = (int)g.blocks.size();
    BlockInfo b;
    b.id = o.block;
    g.blocks.push_back(b);
    g.block_pos[o.block] = bpos;
  } else {
    bpos = it->second;
    if (bpos != (int)g.blocks.size() - 1) IOS_FAIL(IOS_ERR_BLOCK, "block " + std::to_string(o.block) + " is not contiguous");
  }
  BlockInfo& B = g.blocks[bpos];
  if (B.ops.size() >= 64) IOS_FAIL(IOS_ERR_BLOCK, "more than 64 ops in block " + std::to_string(o.block));
  infer_shape(g, o);
  const int local = (int)B.ops.size();
  B.ops.push_back(o.id);
  B.succ.push_back(0);
  B.pred.push_back(0);
  for (int u : o.inputs) {
    if (u == 0) continue;
    if (g.op_block_pos[u] == bpos) {
      B.succ[g.op_local[u]] |= 1ull << local;
      B.pred[local] |= 1ull << g.op_local[u];
    }
  }
  g.ops.push_back(std::move(o));
  g.op_block_pos.push_back(bpos);
  g.op_local.push_back(local);
  *out_op_id = g.ops.back().id;
  ABI_END
}

ios_status ios_graph_num_ops(ios_graph gh, int32_t* n) {
  ABI_BEGIN
  REQUIRE(gh && n, "bad arguments");
  *n = (int32_t)gh->g.ops.size() - 1;
  ABI_END
}

ios_status ios_op_shape(ios_graph gh, int32_t op, int32_t shape[4]) {
  ABI_BEGIN
  REQUIRE(gh && shape && op >= 0 && op < (int)gh->g.ops.size(), "bad arguments");
  const Op& o = gh->g.ops[op];
  shape[0] = o.N;
  shape[1] = o.C;
  shape[2] = o.H;
  shape[3] = o.W;
  ABI_END
}

ios_status ios_graph_num_blocks(ios_graph gh, int32_t* n) {
  ABI_BEGIN
  REQUIRE(gh && n, "bad arguments");
  *n = (int32_t)gh->g.blocks.size();
  ABI_END
}

ios_status ios_graph_block_ops(ios_graph gh, int32_t bp, int32_t* ops, int32_t cap, int32_t* n_ops, int32_t* block_id) {
  ABI_BEGIN
  REQUIRE(gh && n_ops && bp >= 0 && bp < (int)gh->g.blocks.size(), "bad arguments");
  const BlockInfo& b = gh->g.blocks[bp];
  if (ops) {
    REQUIRE(cap >= (int)b.ops.size(), "capacity too small");
    for (size_t i = 0; i < b.ops.size(); ++i) ops[i] = b.ops[i];
  }
  *n_ops = (int32_t)b.ops.size();
  if (block_id) *block_id = b.id;
  ABI_END
}

ios_status ios_stage_mergeable(ios_graph gh, const int32_t* ops, int32_t n, int32_t* m) {
  ABI_BEGIN
  REQUIRE(gh && ops && m && n >= 1, "bad arguments");
  std::vector<int> v(ops, ops + n);
  gh->g.mask_of(v, nullptr);
  *m = gh->g.mergeable(v) ? 1 : 0;
  ABI_END
}

ios_status ios_stage_latency(ios_graph gh, const int32_t* ops, int32_t n, ios_strategy t, const ios_profile_opts* opts,
                             double* out_ms) {
  ABI_BEGIN
  REQUIRE(gh && ops && out_ms && n >= 1, "bad arguments");
  std::vector<int> v(ops, ops + n);
  std::sort(v.begin(), v.end());
  gh->g.mask_of(v, nullptr);
  if (t == IOS_MERGE && !gh->g.mergeable(v)) IOS_FAIL(IOS_ERR_NOT_MERGEABLE, "stage is not mergeable");
  REQUIRE(t == IOS_MERGE || t == IOS_CONCURRENT, "bad strategy");
  *out_ms = stage_latency(gh->g, v, t, opts);
  ABI_END
}

ios_status ios_schedule_dp_ex(ios_graph gh, int32_t r, int32_t s, ios_strategy_set set, ios_cost_fn cost, void* ctx,
                              ios_schedule* out, double* out_cost, int64_t stats[3]) {
  ABI_BEGIN
  REQUIRE(gh && out, "bad arguments");
  REQUIRE(set == IOS_BOTH || set == IOS_MERGE_ONLY || set == IOS_PARALLEL_ONLY, "bad strategy set");
  auto* qh = new ios_schedule_s();
  qh->q.g = &gh->g;
  double c;
  try {
    c = schedule_dp(gh->g, r, s, set, cost, ctx, &qh->q, stats);
  } catch (...) {
    delete qh;
    throw;
  }
  if (out_cost) *out_cost = c;
  *out = qh;
  ABI_END
}

ios_status ios_schedule_refine(ios_graph gh, int32_t r, int32_t s, int32_t reps, double beta_us, ios_schedule* out,
                               int64_t out_stats[4]) {
  ABI_BEGIN
  REQUIRE(gh && out && reps > 0 && beta_us >= 0.0, "bad arguments");
  auto* qh = new ios_schedule_s();
  qh->q.g = &gh->g;
  try {
    schedule_refine(gh->g, r, s, reps, beta_us * 1e-3, &qh->q, out_stats);
    validate_schedule(gh->g, qh->q);
  } catch (...) {
    delete qh;
    throw;
  }
  *out = qh;
  ABI_END
}

ios_status ios_schedule_dp(ios_graph gh, int32_t r, int32_t s, ios_cost_fn cost, void* ctx, ios_schedule* out,
                           double* out_cost) {
  return ios_schedule_dp_ex(gh, r, s, IOS_BOTH, cost, ctx, out, out_cost, nullptr);
}

ios_status ios_schedule_sequential(ios_graph gh, ios_schedule* out) {
  ABI_BEGIN
  REQUIRE(gh && out, "bad arguments");
  auto* qh = new ios_schedule_s();
  qh->q.g = &gh->g;
  for (int v = 1; v < (int)gh->g.ops.size(); ++v) {     // insertion order (Z16)
    Stage st;
    st.ops = {v};
    qh->q.stages.push_back(st);
  }
  *out = qh;
  ABI_END
}

ios_status ios_schedule_greedy(ios_graph gh, ios_schedule* out) {
  ABI_BEGIN
  REQUIRE(gh && out, "bad arguments");
  Graph& g = gh->g;
  auto* qh = new ios_schedule_s();
  qh->q.g = &g;
  for (int bp = 0; bp < (int)g.blocks.size(); ++bp) {   // all ready ops form one stage
    const BlockInfo& b = g.blocks[bp];
    const int n = (int)b.ops.size();
    uint64_t rem = n == 64 ? ~0ull : ((1ull << n) - 1);
    while (rem) {
      uint64_t ready = 0;
      for (int i = 0; i < n; ++i)
        if ((rem >> i & 1) && !(b.pred[i] & rem)) ready |= 1ull << i;
      Stage st;
      st.ops = g.ops_of(bp, ready);
      qh->q.stages.push_back(st);
      rem &= ~ready;
    }
  }
  *out = qh;
  ABI_END
}

ios_status ios_schedule_create(ios_graph gh, int32_t n_stages, const int32_t* sizes, const int32_t* ops,
                               const int32_t* strategies, ios_schedule* out) {
  ABI_BEGIN
  REQUIRE(gh && out && n_stages >= 0 && (n_stages == 0 || (sizes && ops && strategies)), "bad arguments");
  auto* qh = new ios_schedule_s();
  qh->q.g = &gh->g;
  int off = 0;
  for (int i = 0; i < n_stages; ++i) {
    if (sizes[i] < 1) {
      delete qh;
      IOS_FAIL(IOS_ERR_BAD_SCHEDULE, "empty stage");
    }
    Stage st;
    st.ops.assign(ops + off, ops + off + sizes[i]);
    std::sort(st.ops.begin(), st.ops.end());
    st.strategy = strategies[i];
    off += sizes[i];
    qh->q.stages.push_back(st);
  }
  try {
    validate_schedule(gh->g, qh->q);
  } catch (...) {
    delete qh;
    throw;
  }
  *out = qh;
  ABI_END
}

ios_status ios_schedule_num_stages(ios_schedule qh, int32_t* n) {
  ABI_BEGIN
  REQUIRE(qh && n, "bad arguments");
  *n = (int32_t)qh->q.stages.size();
  ABI_END
}

ios_status ios_schedule_stage(ios_schedule qh, int32_t i, int32_t* ops, int32_t cap, int32_t* n_ops, ios_strategy* t,
                              double* latency_ms) {
  ABI_BEGIN
  REQUIRE(qh && n_ops && i >= 0 && i < (int)qh->q.stages.size(), "bad arguments");
  const Stage& st = qh->q.stages[i];
  if (ops) {
    REQUIRE(cap >= (int)st.ops.size(), "capacity too small");
    for (size_t k = 0; k < st.ops.size(); ++k) ops[k] = st.ops[k];
  }
  *n_ops = (int32_t)st.ops.size();
  if (t) *t = (ios_strategy)st.strategy;
  if (latency_ms) *latency_ms = st.latency_ms;
  ABI_END
}

ios_status ios_schedule_tune(ios_graph gh, ios_schedule qh, int32_t trials, int32_t reps) {
  ABI_BEGIN
  REQUIRE(gh && qh, "bad arguments");
  REQUIRE(qh->q.g == &gh->g, "schedule belongs to another graph");
  validate_schedule(gh->g, qh->q);
  tune_schedule(gh->g, qh->q, trials > 0 ? trials : 3, reps > 0 ? reps : 10);
  ABI_END
}

ios_status ios_run(ios_graph gh, ios_schedule qh, const void* d_in, void* d_out, void* stream) {
  ABI_BEGIN
  REQUIRE(gh && qh && d_in && d_out, "bad arguments");
  REQUIRE(qh->q.g == &gh->g, "schedule belongs to another graph");
  validate_schedule(gh->g, qh->q);
  run_schedule(gh->g, qh->q, d_in, d_out, reinterpret_cast<cudaStream_t>(stream));
  ABI_END
}

ios_status ios_run_host(ios_graph gh, ios_schedule qh, const float* h_in, float* h_out, void* stream) {
  ABI_BEGIN
  REQUIRE(gh && qh && h_in && h_out, "bad arguments");
  REQUIRE(qh->q.g == &gh->g, "schedule belongs to another graph");
  Graph& g = gh->g;
  validate_schedule(g, qh->q);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const Op& in = g.ops[0];
  const Op& last = g.ops.back();
  const size_t in_bytes = (size_t)in.N * in.C * in.H * in.W * sizeof(float);
  const size_t out_bytes = (size_t)last.N * last.C * last.H * last.W * sizeof(float);
  IOS_CHECK_CUDA(cudaSetDevice(g.device));
  void *d_in = nullptr, *d_out = nullptr;
  IOS_CHECK_CUDA(cudaMallocAsync(&d_in, in_bytes, st));
  IOS_CHECK_CUDA(cudaMallocAsync(&d_out, out_bytes, st));
  IOS_CHECK_CUDA(cudaMemcpyAsync(d_in, h_in, in_bytes, cudaMemcpyHostToDevice, st));
  run_schedule(g, qh->q, d_in, d_out, st);
  IOS_CHECK_CUDA(cudaMemcpyAsync(h_out, d_out, out_bytes, cudaMemcpyDeviceToHost, st));
  IOS_CHECK_CUDA(cudaFreeAsync(d_in, st));
  IOS_CHECK_CUDA(cudaFreeAsync(d_out, st));
  sync_and_check(g, st);   // IOS_ERR_KERNEL if a dependency wait of this run timed out
  ABI_END
}

ios_status ios_run_timeline(ios_graph gh, ios_schedule qh, const void* d_in, void* d_out, int32_t reps,
                            int32_t l2_flush, double* stage_us, int32_t cap) {
  ABI_BEGIN
  REQUIRE(gh && qh && d_in && d_out && stage_us && reps > 0, "bad arguments");
  REQUIRE(qh->q.g == &gh->g, "schedule belongs to another graph");
  REQUIRE(cap >= 3 * (int)qh->q.stages.size(), "capacity too small (3 doubles per stage)");
  validate_schedule(gh->g, qh->q);
  std::vector<double> v;
  run_timeline(gh->g, qh->q, d_in, d_out, reps, l2_flush != 0, v);
  for (size_t i = 0; i < v.size(); ++i) stage_us[i] = v[i];
  ABI_END
}

ios_status ios_tile_variants_save(ios_graph gh, const char* path) {
  ABI_BEGIN
  REQUIRE(gh && path, "bad arguments");
  save_tile_variants(gh->g, path);
  ABI_END
}

ios_status ios_tile_variants_load(ios_graph gh, const char* path) {
  ABI_BEGIN
  REQUIRE(gh && path, "bad arguments");
  load_tile_variants(gh->g, path);
  ABI_END
}

ios_status ios_sync(ios_graph gh, void* stream) {
  ABI_BEGIN
  REQUIRE(gh, "bad arguments");
  sync_and_check(gh->g, reinterpret_cast<cudaStream_t>(stream));
  ABI_END
}

#ifndef IOS_BUILD_ID
#define IOS_BUILD_ID "unknown"
#endif
const char* ios_build_id(void) { return IOS_BUILD_ID; }

ios_status ios_op_output(ios_graph gh, int32_t op, void* d_out, void* stream) {
  ABI_BEGIN
  REQUIRE(gh && d_out && op >= 0 && op < (int)gh->g.ops.size(), "bad arguments");
  op_output(gh->g, op, d_out, reinterpret_cast<cudaStream_t>(stream));
  ABI_END
}

ios_status ios_schedule_launches(ios_graph gh, ios_schedule qh, int32_t* n) {
  ABI_BEGIN
  REQUIRE(gh && qh && n, "bad arguments");
  validate_schedule(gh->g, qh->q);
  *n = schedule_launches(gh->g, qh->q);
  ABI_END
}

}  // extern "C"

// Latency cache file: one line per measured stage, "block_signature mask strategy ms" (text,
// versioned by the graph signature line so a cache from another graph/math/batch is rejected).
std::string graph_signature(const Graph& g) {
  std::ostringstream s;
  s << "ios-latency-cache v2 batch=" << g.batch << " math=" << (int)g.math << " ops=" << g.ops.size();
  uint64_t h = 1469598103934665603ull;
  for (const Op& o : g.ops) {
    const int f[] = {o.kind, o.block, o.C, o.H, o.W, o.kh, o.kw, o.sh, o.sw, o.ph, o.pw, o.flags, (int)o.inputs.size()};
    for (int v : f) h = (h ^ (uint64_t)(uint32_t)v) * 1099511628211ull;
    for (int u : o.inputs) h = (h ^ (uint64_t)(uint32_t)u) * 1099511628211ull;
  }
  s << " hash=" << std::hex << h;
  return s.str();
}

namespace ios {
void save_latency_cache(const Graph& g, const std::string& path) {
  const std::string tmp = path + ".tmp";
  {
    std::ofstream f(tmp);
    if (!f) IOS_FAIL(IOS_ERR_INVALID_ARG, "cannot write " + path);
    f << graph_signature(g) << "\n";
    f.precision(17);
    // an unsupported stage is cached as inf: written as the token "inf" (istream >> double cannot
    // parse it; the loader reads tokens and converts with strtod, which can)
    for (auto& [k, v] : g.latency_cache) {
      f << std::get<0>(k) << " " << std::get<1>(k) << " " << std::get<2>(k) << " ";
      if (std::isinf(v)) f << "inf";
      else f << v;
      f << "\n";
    }
  }
  std::rename(tmp.c_str(), path.c_str());
}
}  // namespace ios

extern "C" {

ios_status ios_latency_cache_save(ios_graph gh, const char* path) {
  ABI_BEGIN
  REQUIRE(gh && path, "bad arguments");
  save_latency_cache(gh->g, path);
  ABI_END
}

ios_status ios_latency_cache_autosave(ios_graph gh, const char* path) {
  ABI_BEGIN
  REQUIRE(gh, "bad arguments");
  gh->g.cache_autosave = path ? path : "";
  ABI_END
}

ios_status ios_latency_cache_load(ios_graph gh, const char* path) {
  ABI_BEGIN
  REQUIRE(gh && path, "bad arguments");
  std::ifstream f(path);
  if (!f) IOS_FAIL(IOS_ERR_INVALID_ARG, std::string("cannot read ") + path);
  std::string sig;
  std::getline(f, sig);
  if (sig != graph_signature(gh->g)) IOS_FAIL(IOS_ERR_INVALID_ARG, "latency cache belongs to another graph");
  std::string a, b, c, d;
  int line = 1;
  while (f >> a) {
    ++line;
    if (!(f >> b >> c >> d)) IOS_FAIL(IOS_ERR_INVALID_ARG, std::string(path) + ": truncated entry at line " + std::to_string(line));
    char* e1 = nullptr;
    char* e2 = nullptr;
    char* e3 = nullptr;
    char* e4 = nullptr;
    const unsigned long long bsig = std::strtoull(a.c_str(), &e1, 10), m = std::strtoull(b.c_str(), &e2, 10);
    const long t = std::strtol(c.c_str(), &e3, 10);
    const double v = std::strtod(d.c_str(), &e4);
    if (*e1 || *e2 || *e3 || *e4 || (t != IOS_CONCURRENT && t != IOS_MERGE))
      IOS_FAIL(IOS_ERR_INVALID_ARG, std::string(path) + ": malformed entry at line " + std::to_string(line));
    gh->g.latency_cache[std::make_tuple((uint64_t)bsig, (uint64_t)m, (int)t)] = v;
  }
  ABI_END
}

ios_status ios_stage_trace(ios_graph gh, const int32_t* ops, int32_t n, ios_strategy t, uint64_t* out, int32_t cap,
                           int32_t* grid) {
  ABI_BEGIN
  REQUIRE(gh && ops && out && grid && n >= 1, "bad arguments");
  std::vector<int> v(ops, ops + n);
  std::sort(v.begin(), v.end());
  *grid = stage_trace(gh->g, v, t, out, cap);
  ABI_END
}

void ios_schedule_destroy(ios_schedule q) { delete q; }
void ios_graph_destroy(ios_graph g) { delete g; }

}  // extern "C"
