// Internal host-side structures of libios (not part of the ABI; see include/ios.h).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <memory>
#include <string>
#include <tuple>
#include <unordered_map>
#include <vector>

#include "../../include/ios.h"
#include "stage_desc.h"

namespace ios {

// ------------------------------------------------------------------------------------ errors
struct Error {
  ios_status code;
  std::string msg;
};
void set_error(const std::string& msg);
#define IOS_FAIL(code, msg) throw ::ios::Error{(code), (msg)}
#define IOS_CHECK_CUDA(expr)                                                                    \
  do {                                                                                          \
    cudaError_t e_ = (expr);                                                                    \
    if (e_ != cudaSuccess)                                                                      \
      IOS_FAIL(e_ == cudaErrorMemoryAllocation ? IOS_ERR_OOM : IOS_ERR_CUDA,                    \
               std::string(#expr) + ": " + cudaGetErrorString(e_));                             \
  } while (0)

// ------------------------------------------------------------------------------------ graph
struct Op {
  int id = 0;
  int kind = 0;      // ios_op_kind
  int block = 0;
  int cout = 0, kh = 1, kw = 1, sh = 1, sw = 1, ph = 0, pw = 0, flags = 0;
  std::vector<int> inputs;
  std::vector<float> weight, bias, add_w;
  int N = 0, C = 0, H = 0, W = 0;   // output shape (logical channels)
  int Cp = 0;                        // padded channels (multiple of 8)
  std::string name;
};

struct BlockInfo {
  int id = 0;
  std::vector<int> ops;            // global ids, insertion order; bit i of a mask = ops[i]
  std::vector<uint64_t> succ, pred;  // within-block adjacency masks
};

struct StagePlan;  // device.cpp

struct DeviceState;  // device.cpp

struct Graph {
  int batch = 1, c = 0, h = 0, w = 0;
  ios_math math = IOS_MATH_TF32;
  int device = 0;
  std::vector<Op> ops;                       // ops[0] = graph input
  std::vector<BlockInfo> blocks;
  std::unordered_map<int, int> block_pos;    // block id -> index in `blocks`
  std::vector<int> op_block_pos, op_local;   // per op: block position, local index
  // stage-latency cache: key (block signature, mask, strategy); identical blocks (e.g. repeated
  // NASNet cells) share their measurements
  std::map<std::tuple<uint64_t, uint64_t, int>, double> latency_cache;
  std::vector<uint64_t> block_sigs;   // lazily computed
  std::string cache_autosave;         // checkpoint the latency cache here after each block's search
  uint64_t block_sig(int bpos);
  DeviceState* dev = nullptr;
  ~Graph();

  int dtype() const { return math == IOS_MATH_BF16 ? ET_BF16 : math == IOS_MATH_FP32_SIMT ? ET_F32X : ET_F32; }
  int esize() const { return math == IOS_MATH_BF16 ? 2 : 4; }
  // stage helpers
  uint64_t mask_of(const std::vector<int>& ops, int* bpos) const;   // throws NOT_A_STAGE
  std::vector<int> ops_of(int bpos, uint64_t mask) const;
  bool mergeable(const std::vector<int>& ops) const;
  std::vector<uint64_t> components(int bpos, uint64_t mask) const;
};

struct Stage {
  std::vector<int> ops;   // global ids, ascending
  int strategy = IOS_CONCURRENT;
  double latency_ms = -1.0;
};

struct Schedule {
  std::vector<Stage> stages;
  Graph* g = nullptr;
  // execution cache (device.cpp)
  cudaGraphExec_t exec = nullptr;
  cudaGraph_t graph = nullptr;
  const void* exec_in = nullptr;
  void* exec_out = nullptr;
  cudaStream_t exec_stream = nullptr;
  uint64_t exec_gen = 0;   // DeviceState::plan_gen the exec was captured with
  int n_launches = -1;
  ~Schedule();
};

void validate_schedule(const Graph& g, const Schedule& q);   // throws BAD_SCHEDULE / NOT_MERGEABLE
void save_latency_cache(const Graph& g, const std::string& path);

// ------------------------------------------------------------------------------------ device
double stage_latency(Graph& g, const std::vector<int>& ops, int strategy, const ios_profile_opts* opts);
// Batch measurement for the DP's search (fills g.latency_cache for every (mask, strategy) of block bpos)
void measure_stages(Graph& g, int bpos, const std::vector<std::pair<uint64_t, int>>& stages);
void run_schedule(Graph& g, Schedule& q, const void* d_in, void* d_out, cudaStream_t st);
void op_output(Graph& g, int op, void* d_out, cudaStream_t st);
int schedule_launches(Graph& g, Schedule& q);
void save_tile_variants(Graph& g, const std::string& path);
void load_tile_variants(Graph& g, const std::string& path);
void run_timeline(Graph& g, Schedule& q, const void* d_in, void* d_out, int reps, bool flush, std::vector<double>& out);
int stage_trace(Graph& g, const std::vector<int>& ops, int strategy, uint64_t* out, int cap);
void destroy_device(Graph& g);
void tune_schedule(Graph& g, Schedule& q, int trials, int reps);
double schedule_dp(Graph& g, int r, int s, int set, ios_cost_fn cost, void* ctx, Schedule* out, int64_t stats[3],
                   double stage_bias_ms = 0.0);
void schedule_refine(Graph& g, int r, int s, int reps, double beta_ms, Schedule* out, int64_t stats[4]);
void destroy_schedule_exec(Schedule& q);
void sync_and_check(Graph& g, cudaStream_t st);   // synchronise, then IOS_ERR_KERNEL if a wait timed out

// kernels (stage_kernel.cu)
cudaError_t launch_stage(const StageDesc& sd, int dtype, int grid, cudaStream_t st);
int stage_cluster_ctas();   // co-resident CTAs of a cluster-split-K launch (clusters of kClusterCtas); 0 on error
cudaError_t launch_nchw_to_nhwc(const float* in, const View& out, int dtype, int N, int C, cudaStream_t st);
cudaError_t launch_nchw_unfold(const float* in, const View& out, int dtype, int N, int C, int W, int kw, int sw, int pw,
                               cudaStream_t st);
cudaError_t launch_nhwc_to_nchw(const View& in, int dtype, float* out, int N, int C, cudaStream_t st);
cudaError_t launch_l2_flush(void* buf, int64_t bytes, cudaStream_t st);

inline int popcount64(uint64_t m) { return __builtin_popcountll(m); }
inline int round_up(int x, int m) { return (x + m - 1) / m * m; }

}  // namespace ios
