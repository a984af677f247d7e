// Graph construction, shape inference, blocks, merge legality, schedule objects and the C-ABI
// entry points that do not touch the device. P:n = /root/reference/PAPER.md line n.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <sstream>
#include <algorithm>

#include "ios_core.h"

namespace ios {

static thread_local std::string g_last_error;
void set_error(const std::string& msg) { g_last_error = msg; }

Graph::~Graph() { destroy_device(*this); }
Schedule::~Schedule() { destroy_schedule_exec(*this); }

static int pool_out(int h, int k, int s, int p, bool ceil_mode) {
  // torch rule (Z11): with ceil_mode the last window must start inside the input or the
  // left padding.
  if (!ceil_mode) return (h + 2 * p - k) / s + 1;
  int o = (h + 2 * p - k + s - 1) / s + 1;
  if ((o - 1) * s >= h + p) --o;
  return o;
}

uint64_t Graph::mask_of(const std::vector<int>& ids, int* bpos) const {
  if (ids.empty()) IOS_FAIL(IOS_ERR_NOT_A_STAGE, "empty stage");
  uint64_t m = 0;
  int bp = -1;
  for (int v : ids) {
    if (v < 1 || v >= (int)ops.size()) IOS_FAIL(IOS_ERR_NOT_A_STAGE, "stage names an unknown op " + std::to_string(v));
    if (bp >= 0 && op_block_pos[v] != bp) IOS_FAIL(IOS_ERR_NOT_A_STAGE, "stage spans blocks");
    bp = op_block_pos[v];
    const uint64_t bit = 1ull << op_local[v];
    if (m & bit) IOS_FAIL(IOS_ERR_NOT_A_STAGE, "op repeated in a stage");
    m |= bit;
  }
  if (bpos) *bpos = bp;
  return m;
}

std::vector<int> Graph::ops_of(int bpos, uint64_t mask) const {
  std::vector<int> r;
  const BlockInfo& b = blocks[bpos];
  for (size_t i = 0; i < b.ops.size(); ++i)
    if (mask >> i & 1) r.push_back(b.ops[i]);
  return r;
}

// Operator merge legality (Z4): plain convolutions reading the identical
// input tensor, same stride and pre-ReLU, equal output H x W, at least two of them.
bool Graph::mergeable(const std::vector<int>& ids) const {
  if (ids.size() < 2) return false;
  const Op& f = ops[ids[0]];
  for (int v : ids) {
    const Op& o = ops[v];
    if (o.kind != IOS_OP_CONV) return false;
    if (o.inputs[0] != f.inputs[0] || o.sh != f.sh || o.sw != f.sw) return false;
    if ((o.flags & IOS_F_RELU_PRE) != (f.flags & IOS_F_RELU_PRE)) return false;
    if (o.H != f.H || o.W != f.W) return false;
  }
  return true;
}

// Groups = connected components of the undirected subgraph induced by the stage (Z3).
std::vector<uint64_t> Graph::components(int bpos, uint64_t mask) const {
  const BlockInfo& b = blocks[bpos];
  std::vector<uint64_t> comps;
  uint64_t left = mask;
  while (left) {
    const int i = __builtin_ctzll(left);
    uint64_t comp = 1ull << i, frontier = comp;
    while (frontier) {
      const int u = __builtin_ctzll(frontier);
      frontier &= frontier - 1;
      const uint64_t nb = (b.succ[u] | b.pred[u]) & mask & ~comp;
      comp |= nb;
      frontier |= nb;
    }
    comps.push_back(comp);
    left &= ~comp;
  }
  return comps;
}

// A schedule is valid iff every op appears once, stages lie in one block, blocks run in order and
// every edge (u, v) goes to a later stage or stays inside one concurrent stage (then u and v share
// a group and run in insertion order) — i.e. each stage is an ending of the remaining ops.
void validate_schedule(const Graph& g, const Schedule& q) {
  const int n = (int)g.ops.size() - 1;
  std::vector<int> stage_of(n + 1, -1);
  int last_bpos = -1;
  for (size_t si = 0; si < q.stages.size(); ++si) {
    const Stage& st = q.stages[si];
    int bpos = -1;
    g.mask_of(st.ops, &bpos);
    if (bpos < last_bpos) IOS_FAIL(IOS_ERR_BAD_SCHEDULE, "blocks out of order");
    last_bpos = bpos;
    for (int v : st.ops) {
      if (stage_of[v] >= 0) IOS_FAIL(IOS_ERR_BAD_SCHEDULE, "op " + std::to_string(v) + " scheduled twice");
      stage_of[v] = (int)si;
    }
    if (st.strategy == IOS_MERGE && !g.mergeable(st.ops))
      IOS_FAIL(IOS_ERR_NOT_MERGEABLE, "merge stage is not mergeable");
    if (st.strategy != IOS_MERGE && st.strategy != IOS_CONCURRENT) IOS_FAIL(IOS_ERR_INVALID_ARG, "bad strategy");
  }
  for (int v = 1; v <= n; ++v)
    if (stage_of[v] < 0) IOS_FAIL(IOS_ERR_BAD_SCHEDULE, "op " + std::to_string(v) + " not scheduled");
  for (int v = 1; v <= n; ++v)
    for (int u : g.ops[v].inputs) {
      if (u == 0) continue;
      const int su = stage_of[u], sv = stage_of[v];
      if (su > sv || (su == sv && q.stages[su].strategy == IOS_MERGE))
        IOS_FAIL(IOS_ERR_BAD_SCHEDULE, "edge " + std::to_string(u) + "->" + std::to_string(v) + " violates the stage order");
    }
}

// Structural hash of a block: op kinds, hyper-parameters, output shapes, in-block edges (as local
// indices) and the shapes of external inputs. Stage latency depends on these, not on weights.
uint64_t Graph::block_sig(int bpos) {
  if (block_sigs.size() != blocks.size()) block_sigs.assign(blocks.size(), 0);
  if (block_sigs[bpos]) return block_sigs[bpos];
  uint64_t h = 1469598103934665603ull;
  auto mix = [&](int64_t v) { h = (h ^ (uint64_t)v) * 1099511628211ull; };
  mix(batch);
  mix((int)math);
  for (int v : blocks[bpos].ops) {
    const Op& o = ops[v];
    for (int64_t x : {(int64_t)o.kind, (int64_t)o.C, (int64_t)o.H, (int64_t)o.W, (int64_t)o.kh, (int64_t)o.kw,
                      (int64_t)o.sh, (int64_t)o.sw, (int64_t)o.ph, (int64_t)o.pw, (int64_t)o.flags,
                      (int64_t)o.inputs.size()})
      mix(x);
    for (int u : o.inputs) {
      if (u != 0 && op_block_pos[u] == bpos) {
        mix(1000000 + op_local[u]);
      } else {
        mix(ops[u].C);
        mix(ops[u].H);
        mix(ops[u].W);
      }
    }
  }
  if (h == 0) h = 1;
  block_sigs[bpos] = h;
  return h;
}

int pool_out_size(int h, int k, int s, int p, bool ceil_mode) { return pool_out(h, k, s, p, ceil_mode); }
const char* last_error_cstr() { return g_last_error.c_str(); }

}  // namespace ios
