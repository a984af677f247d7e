// Device side of libios: activation memory plan (concat elision), weight packing, stage planning
// (tile scheduler inputs), the CUDA-event stage profiler and the CUDA-graph runner.
//
//   stage plan: problems + tiles + dependency counters for one (block, mask, T)
//   profiler    (A7, "directly measures the latencies"): W warm-up launches, then trials of R
//               back-to-back launches between CUDA events; the median trial mean (Z15)
//   runner      (A9): the stages of Q in order, captured once into a CUDA graph
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <limits>
#include <sstream>

#include <cuda.h>

#include "ios_core.h"

namespace ios {

namespace {

constexpr double kInf = std::numeric_limits<double>::infinity();

struct OpDev {
  View out{};                 // where the op's output lives (possibly a slice of a concat buffer)
  bool elided = false;        // concat/identity realised by addressing alone
  int alias_parent = -1;      // concat this op's output is a slice of
  int alias_off = 0;          // channel offset inside the parent
  void* wpack = nullptr;      // packed GEMM weights (conv / linear / sepconv pointwise)
  int wpack_n8 = 0;           // packed rows (multiple of 8)
  float* bias = nullptr;      // fp32, zero padded
  float* dw = nullptr;        // sepconv depthwise weights fp32, tap-major [kh*kw][Cp_in]
  float* dwc = nullptr;       // the same, chunk-major [Cp_in / elems][kh*kw][elems] (fused halo path)
  float* add_w = nullptr;     // add / sepconv aggregation weights
  View dw_out{};              // sepconv depthwise scratch (NHWC, Cp_in channels)
  int tt = 0, kblk = 0;       // weights packed for the tap-TMA im2col path (K = taps x kblk blocks)
  int unfold = 0;             // reads the W-unfolded graph input (DeviceState::unfold): kernel kh x 1
};

}  // namespace

struct StagePlan {
  StageDesc sd{};
  int grid = 0;
  int dtype = 0;
  bool empty = true;
  void* dmem = nullptr;       // problems | views | segments
  int* counters = nullptr;
  void* workspace = nullptr;
  void* merged_pack = nullptr;
  float* merged_bias = nullptr;
  std::vector<void*> allocs;  // pool allocations owned by this plan
};

struct DeviceState {
  bool ready = false;
  int num_sms = 148;
  int cluster_ctas = 0;              // co-resident CTAs of a cluster-split-K launch (stage_cluster_ctas)
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  std::vector<OpDev> od;
  std::vector<void*> allocs;
  int* err = nullptr;                // kernel error flag: pinned, host-mapped (read without a copy)
  void* l2buf = nullptr;
  int64_t l2bytes = 0;
  std::map<std::tuple<int, uint64_t, int>, StagePlan*> plans;
  // per-stage tiling variant chosen by ios_schedule_tune (absent = 0, the default knobs)
  std::map<std::tuple<int, uint64_t, int>, int> tile_variant;
  std::vector<StagePlan*> retired;   // plans replaced by tuning (a captured schedule may use them)
  uint64_t plan_gen = 0;             // bumped when tuning replaces plans: captured schedules re-capture
  // W-unfolded copy of the graph input for a narrow first conv (Cin*esz < 64 B, kw > 1): pixel
  // (n, h, ow) holds the kw input pixels the conv's output column ow reads along W, channel
  // j * C + c = x[n, h, ow*sw - pw + j, c] (zero outside), padded to one 128 B block. The conv then
  // runs as a kh x 1 conv with stride (sh, 1) on the tap-TMA path: dense 128 B taps instead of a
  // 16 B-granular gather (measured: SqueezeNet conv1 7x7/2 at batch 128 was 37 % of the network).
  bool unfold = false;
  View unfold_view{};
  int unfold_kw = 0, unfold_sw = 1, unfold_pw = 0;
};

namespace {

// Persistent graph memory (activations, weights) is cudaMalloc'ed and lives with the graph.
// Stage-plan memory (`owner` != nullptr) comes from the stream-ordered pool so the profiler can
// build, measure and drop hundreds of thousands of candidate stages cheaply.
void* dmalloc(DeviceState& d, size_t bytes, std::vector<void*>* owner = nullptr) {
  void* p = nullptr;
  bytes = std::max<size_t>(bytes, 256);
  if (owner) {
    IOS_CHECK_CUDA(cudaMallocAsync(&p, bytes, d.stream));
    IOS_CHECK_CUDA(cudaMemsetAsync(p, 0, bytes, d.stream));
    owner->push_back(p);
  } else {
    IOS_CHECK_CUDA(cudaMalloc(&p, bytes));
    IOS_CHECK_CUDA(cudaMemset(p, 0, bytes));
    d.allocs.push_back(p);
  }
  return p;
}

template <class T>
T* upload(DeviceState& d, const std::vector<T>& v, size_t min_elems = 0, std::vector<void*>* owner = nullptr) {
  const size_t n = std::max(v.size(), min_elems);
  T* p = static_cast<T*>(dmalloc(d, n * sizeof(T), owner));
  if (!v.empty()) {
    if (owner)
      IOS_CHECK_CUDA(cudaMemcpyAsync(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, d.stream));
    else
      IOS_CHECK_CUDA(cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
  }
  return p;
}

uint32_t tf32_rne_bits(float x) {
  uint32_t u;
  std::memcpy(&u, &x, 4);
  if ((u & 0x7F800000u) == 0x7F800000u) return u;   // inf / nan
  u += 0xFFFu + ((u >> 13) & 1u);
  return u & ~0x1FFFu;
}
uint16_t bf16_rne_bits(float x) {
  uint32_t u;
  std::memcpy(&u, &x, 4);
  if ((u & 0x7F800000u) == 0x7F800000u) return (uint16_t)(u >> 16);
  u += 0x7FFFu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

// Packs a GEMM weight matrix w(n, k), n < N, k < K, into the UMMA K-major SWIZZLE_NONE smem image
// order: [k chunk][n / 8][8 pieces of 16 B][n % 8][16 B]. Any BN rows starting at a multiple of 8
// of one chunk are then one contiguous run of BN * 128 bytes (one cp.async.bulk).
template <class F>
void* pack_gemm(DeviceState& d, int N, int K, int dtype, F w, int* n8_out, std::vector<void*>* owner = nullptr) {
  // dtype: ET_F32 -> TF32-rounded (RNE) fp32, ET_BF16 -> bf16 (RNE), ET_F32X -> exact fp32
  const bool bf16 = dtype == ET_BF16;
  const int esz = bf16 ? 2 : 4, elems = kChunkBytes / esz, vec = 16 / esz;
  const int kch = (K + elems - 1) / elems;
  const int n8 = round_up(N, 8);
  std::vector<uint8_t> buf((size_t)kch * n8 * kChunkBytes, 0);
  for (int n = 0; n < N; ++n) {
    for (int k = 0; k < K; ++k) {
      const float v = w(n, k);
      if (v == 0.0f) continue;
      const int c = k / elems, kk = k % elems, pc = kk / vec, e = kk % vec;
      const size_t off = (((size_t)c * (n8 / 8) + n / 8) * 8 + pc) * 128 + (n % 8) * 16 + e * esz;
      if (bf16) {
        const uint16_t b = bf16_rne_bits(v);
        std::memcpy(&buf[off], &b, 2);
      } else if (dtype == ET_F32X) {
        std::memcpy(&buf[off], &v, 4);                 // exact fp32 (CUDA-core FMA path)
      } else {
        const uint32_t b = tf32_rne_bits(v);
        std::memcpy(&buf[off], &b, 4);
      }
    }
  }
  *n8_out = n8;
  return upload(d, buf, 0, owner);
}

int64_t view_elems(const Op& o, int C) { return (int64_t)o.N * o.H * o.W * C; }

// Output patch of one tap-TMA M tile: tN images x tR rows x tWt columns (<= 128 pixels, TMA box
// dims <= 256 input elements). Whole images when everything fits one tile (the swap-AB case: the
// tile row is then the pixel index); otherwise the (tWt, tR) with the fewest tiles.
struct TTGeom {
  int tN = 0, tR = 0, tWt = 0, tiles_h = 0, tiles_w = 0, tiles = 0;
};
TTGeom tt_geometry(int batch, int Ho, int Wo, int sh, int sw) {
  TTGeom best;
  if ((int64_t)batch * Ho * Wo <= kBM && Wo * sw <= 256 && Ho * sh <= 256) {
    best.tN = batch; best.tR = Ho; best.tWt = Wo;
    best.tiles_h = best.tiles_w = best.tiles = 1;
    return best;
  }
  for (int wt = std::min(Wo, kBM); wt >= 1; --wt) {
    if (wt * sw > 256) continue;
    const int r = std::min(std::min(Ho, kBM / wt), 256 / sh);
    if (r < 1) continue;
    const int tn = (r == Ho && wt == Wo) ? std::max(1, std::min(batch, kBM / (Ho * Wo))) : 1;
    const int th = (Ho + r - 1) / r, tw = (Wo + wt - 1) / wt;
    const int tiles = ((batch + tn - 1) / tn) * th * tw;
    if (best.tiles == 0 || tiles < best.tiles) {
      best.tN = tn; best.tR = r; best.tWt = wt;
      best.tiles_h = th; best.tiles_w = tw; best.tiles = tiles;
    }
  }
  return best;
}

// Fused Relu-SepConv patch tiles: at most 16 quads (QW adjacent columns) per tile, so each of the
// 128 producer threads computes ONE (quad, 16 B piece) item per K chunk: the depthwise half is
// latency-bound (dependent load rounds per item), so parallelism across CTAs beats M-tile fill
// (the MMA is idle most of the time anyway). Fewest tiles wins.
TTGeom fdw_geometry(int batch, int Ho, int Wo, int qw) {
  constexpr int kQuads = 16;
  TTGeom best;
  for (int wt = std::min(Wo, kQuads * qw); wt >= 1; --wt) {
    const int qpr = (wt + qw - 1) / qw;             // quads per patch row
    const int r = std::max(1, std::min(Ho, kQuads / qpr));
    const int tn = (r == Ho && wt == Wo) ? std::max(1, std::min(batch, kQuads / (qpr * Ho))) : 1;
    const int th = (Ho + r - 1) / r, tw = (Wo + wt - 1) / wt;
    const int tiles = ((batch + tn - 1) / tn) * th * tw;
    if (best.tiles == 0 || tiles < best.tiles) {
      best.tN = tn; best.tR = r; best.tWt = wt;
      best.tiles_h = th; best.tiles_w = tw; best.tiles = tiles;
    }
  }
  return best;
}

// Tap-TMA im2col eligibility: returns the number of 128 B channel blocks per tap (0 = use the
// cp.async gather or the 2D TMA path). Pre-ReLU convs need the gather (the ReLU is applied on the
// way to smem); 1x1/s1/unpadded convs take the plain 2D TMA; narrow inputs would pad K too much;
// patch tiles must not waste much more M than the gather's dense 128-pixel tiles.
bool tap_tma_enabled();
int tap_tma_blocks(const Graph& g, int cin_p, int kh, int kw, int sh, int sw, int ph, int pw, int flags, int batch,
                   int Ho, int Wo) {
  if (g.math == IOS_MATH_FP32_SIMT || (flags & IOS_F_RELU_PRE)) return 0;
  if (!tap_tma_enabled()) return 0;
  if (kh == 1 && kw == 1 && sh == 1 && sw == 1 && ph == 0 && pw == 0) return 0;
  if (sh > 8 || sw > 8) return 0;
  const int elems = kChunkBytes / g.esize();
  const int kblk = (cin_p + elems - 1) / elems;
  // at most 1.5x K padding by default (IOS_TT_PAD2 = twice the allowed ratio: 3 -> 1.5x, 4 -> 2x)
  static const int pad2 = getenv("IOS_TT_PAD2") ? atoi(getenv("IOS_TT_PAD2")) : 3;
  if (cin_p < 16 || kblk * elems * 2 > cin_p * pad2) return 0;
  const int64_t dense = ((int64_t)batch * Ho * Wo + kBM - 1) / kBM;
  if ((int64_t)tt_geometry(batch, Ho, Wo, sh, sw).tiles * 4 > dense * 5) return 0;
  return kblk;
}

void ensure_device(Graph& g) {
  if (g.dev && g.dev->ready) return;
  if (!g.dev) g.dev = new DeviceState();
  DeviceState& d = *g.dev;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= g.device)
    IOS_FAIL(IOS_ERR_CUDA, "no CUDA device " + std::to_string(g.device) + " (the engine has no CPU fallback)");
  IOS_CHECK_CUDA(cudaSetDevice(g.device));
  cudaDeviceProp prop;
  IOS_CHECK_CUDA(cudaGetDeviceProperties(&prop, g.device));
  if (prop.major != 10 || prop.minor != 0)
    IOS_FAIL(IOS_ERR_CUDA, std::string("libios is built for sm_100a; device is ") + prop.name);
  d.num_sms = prop.multiProcessorCount;
  d.cluster_ctas = stage_cluster_ctas() / kClusterCtas * kClusterCtas;
  IOS_CHECK_CUDA(cudaStreamCreateWithFlags(&d.stream, cudaStreamNonBlocking));
  {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, g.device) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  }
  IOS_CHECK_CUDA(cudaEventCreate(&d.ev0));
  IOS_CHECK_CUDA(cudaEventCreate(&d.ev1));
  {
    void* p = nullptr;
    IOS_CHECK_CUDA(cudaHostAlloc(&p, 64, cudaHostAllocMapped | cudaHostAllocPortable));
    std::memset(p, 0, 64);
    void* dp = nullptr;
    IOS_CHECK_CUDA(cudaHostGetDevicePointer(&dp, p, 0));
    if (dp != p) {
      cudaFreeHost(p);
      IOS_FAIL(IOS_ERR_CUDA, "host-mapped error flag needs unified addressing");
    }
    d.err = static_cast<int*>(p);
  }
  d.l2bytes = 2 * (int64_t)prop.l2CacheSize;

  const int n = (int)g.ops.size();
  d.od.assign(n, OpDev{});
  // ---- concat elision: producers write straight into channel slices of the concat's buffer.
  // Outer (later) concats first, so nested concats resolve top-down.
  for (int v = n - 1; v >= 1; --v) {
    const Op& o = g.ops[v];
    if (o.kind != IOS_OP_CONCAT) continue;
    bool ok = true;
    for (size_t i = 0; i < o.inputs.size() && ok; ++i) {
      const int u = o.inputs[i];
      if (u == 0 || d.od[u].alias_parent >= 0 || g.ops[u].C % 8 != 0) ok = false;
      for (size_t j = 0; j < i; ++j)
        if (o.inputs[j] == u) ok = false;
    }
    if (!ok) continue;
    int off = 0;
    for (int u : o.inputs) {
      d.od[u].alias_parent = v;
      d.od[u].alias_off = off;
      off += g.ops[u].C;
    }
    d.od[v].elided = true;
  }
  // ---- allocate root buffers, then resolve views top-down (parents have larger ids)
  for (int v = 0; v < n; ++v) {
    if (d.od[v].alias_parent >= 0) continue;
    const Op& o = g.ops[v];
    void* p = dmalloc(d, view_elems(o, o.Cp) * g.esize());
    d.od[v].out = View{(uint64_t)p, o.Cp, 0, o.Cp, o.C, o.H, o.W};
  }
  for (int v = n - 1; v >= 0; --v) {
    if (d.od[v].alias_parent < 0) continue;
    // parents are resolved first because they have larger ids and we walk downwards
    const View& pv = d.od[d.od[v].alias_parent].out;
    const Op& o = g.ops[v];
    d.od[v].out = View{pv.ptr, pv.cstride, pv.coff + d.od[v].alias_off, o.Cp, o.C, o.H, o.W};
  }
  // identities not written into a concat are pure aliases of their input
  for (int v = 1; v < n; ++v) {
    const Op& o = g.ops[v];
    if (o.kind == IOS_OP_IDENTITY && d.od[v].alias_parent < 0) {
      d.od[v].out = d.od[o.inputs[0]].out;
      d.od[v].elided = true;
    }
  }
  // ---- W-unfolded graph input (at most one narrow first conv may use it; others read op 0 as is)
  {
    static const bool on = !getenv("IOS_UNFOLD") || atoi(getenv("IOS_UNFOLD")) != 0;
    const int elems = kChunkBytes / g.esize();
    for (int v = 1; v < n && on && g.math != IOS_MATH_FP32_SIMT; ++v) {
      const Op& o = g.ops[v];
      const Op& x = g.ops[0];
      if (o.kind != IOS_OP_CONV || o.inputs[0] != 0 || (o.flags & IOS_F_RELU_PRE)) continue;
      if (x.Cp * g.esize() >= 64 || o.kw < 2 || o.sw > o.kw || o.kw * x.C > elems) continue;
      // worth its extra layout launch only for large outputs (measured at batch 1, Inception V3's
      // 149x149 stem conv: +0.3 % end to end; SqueezeNet conv1 at batch 128: 984 -> 332 us)
      if ((int64_t)o.N * o.H * o.W < 65536) continue;
      void* p = dmalloc(d, (size_t)x.N * x.H * o.W * elems * g.esize());
      d.unfold = true;
      d.unfold_view = View{(uint64_t)p, elems, 0, elems, o.kw * x.C, x.H, o.W};
      d.unfold_kw = o.kw;
      d.unfold_sw = o.sw;
      d.unfold_pw = o.pw;
      d.od[v].unfold = 1;
      break;
    }
  }
  // ---- weights
  const int wdt = g.dtype();
  for (int v = 1; v < n; ++v) {
    const Op& o = g.ops[v];
    OpDev& e = d.od[v];
    const Op& x = g.ops[o.inputs[0]];
    if (!o.add_w.empty()) e.add_w = upload(d, o.add_w);
    if (o.kind == IOS_OP_CONV && e.unfold) {
      // kh x 1 conv over the unfolded input: K = kh taps x one 128 B block, channel j * C + c of
      // tap i holds W[co][c][i][j]
      const int cin = x.C, kh = o.kh, kw = o.kw, elems = kChunkBytes / g.esize();
      const float* W = o.weight.data();
      e.kblk = 1;
      e.tt = 1;
      e.wpack = pack_gemm(d, o.Cp, kh * elems, wdt, [&](int nn, int k) -> float {
        if (nn >= o.cout) return 0.0f;
        const int i = k / elems, ch = k % elems;
        if (ch >= kw * cin) return 0.0f;
        const int j = ch / cin, c = ch % cin;
        return W[(((size_t)nn * cin + c) * kh + i) * kw + j];
      }, &e.wpack_n8);
      std::vector<float> b(o.bias);
      e.bias = upload(d, b, (size_t)round_up(o.Cp, 256) + 16);
    } else if (o.kind == IOS_OP_CONV || o.kind == IOS_OP_LINEAR) {
      const int cin = x.C, cin_p = x.Cp, kh = o.kh, kw = o.kw;
      const float* W = o.weight.data();
      // tap-TMA im2col packs K per tap in whole 128 B channel blocks (zero rows for the padding)
      e.kblk = o.kind == IOS_OP_CONV ? tap_tma_blocks(g, cin_p, kh, kw, o.sh, o.sw, o.ph, o.pw, o.flags, g.batch, o.H, o.W)
                                     : 0;
      e.tt = e.kblk > 0;
      const int tapk = e.tt ? e.kblk * (kChunkBytes / g.esize()) : cin_p;
      e.wpack = pack_gemm(d, o.Cp, kh * kw * tapk, wdt, [&](int nn, int k) -> float {
        if (nn >= o.cout) return 0.0f;
        const int tap = k / tapk, ci = k % tapk;
        if (ci >= cin) return 0.0f;
        const int i = tap / kw, j = tap % kw;
        return W[(((size_t)nn * cin + ci) * kh + i) * kw + j];
      }, &e.wpack_n8);
      std::vector<float> b(o.bias);
      e.bias = upload(d, b, (size_t)round_up(o.Cp, 256) + 16);
    } else if (o.kind == IOS_OP_SEPCONV) {
      const int c = x.C, cp = x.Cp, kk = o.kh * o.kw;
      // tap-major [kh*kw][Cp]: a 16 B vector of consecutive channels per tap
      std::vector<float> dw((size_t)cp * kk, 0.0f);
      for (int ch = 0; ch < c; ++ch)
        for (int t = 0; t < kk; ++t) dw[(size_t)t * cp + ch] = o.weight[(size_t)ch * kk + t];
      e.dw = upload(d, dw);
      {
        const int el = kChunkBytes / g.esize(), nch = (cp + el - 1) / el;
        std::vector<float> dwc((size_t)nch * kk * el, 0.0f);
        for (int ch = 0; ch < c; ++ch)
          for (int t = 0; t < kk; ++t) dwc[((size_t)(ch / el) * kk + t) * el + ch % el] = o.weight[(size_t)ch * kk + t];
        e.dwc = upload(d, dwc);
      }
      const float* PW = o.weight.data() + (size_t)c * kk;
      e.wpack = pack_gemm(d, o.Cp, cp, wdt, [&](int nn, int k) -> float {
        return (nn < o.cout && k < c) ? PW[(size_t)nn * c + k] : 0.0f;
      }, &e.wpack_n8);
      std::vector<float> b(o.bias);
      e.bias = upload(d, b, (size_t)round_up(o.Cp, 256) + 16);
      void* p = dmalloc(d, (size_t)o.N * o.H * o.W * cp * g.esize());
      e.dw_out = View{(uint64_t)p, cp, 0, cp, c, o.H, o.W};
    }
  }
  d.ready = true;
}

// ------------------------------------------------------------------------------ stage planning
struct GemmSpec {
  int M, N16, K, kch, Npad8;
  int BN, ntn, mt, split, cps;
  int swap;   // swap-AB: weights are the 128-row MMA operand, the (<= 128) pixels are N
  int max_bn = kMaxBN;
  int tt_tiles = 0;   // tap-TMA: number of patch M tiles (0 = dense 128-pixel tiles)
  int fdw = 0;        // fused Relu-SepConv (1 register form: split K down to one chunk; 2 halo form:
                      // never split K, the CTA pipelines its chunks); never narrow N (each N tile
                      // would recompute the depthwise half)
  double chunk_cost = 1.0;   // relative cost of one K chunk (fused depthwise chunks are compute)
};

// Fused Relu-SepConv eligibility: square window k in {3, 5, 7}, stride 1-2, at most
// 8 aggregated inputs, tcgen05 math modes (FP32-SIMT keeps the two-problem form)
TTGeom halo_geometry(int batch, int Ho, int Wo, int k, int s, int qw);
bool fuse_dw_ok(const Graph& g, const Op& o) {
  static const bool on = [] {
    const char* v = getenv("IOS_FUSE_DW");
    return v ? atoi(v) != 0 : true;
  }();
  if (!on || g.math == IOS_MATH_FP32_SIMT) return false;
  if (o.kh != o.kw || o.sh != o.sw || o.ph != o.pw) return false;
  if (!(o.kh == 3 || o.kh == 5 || o.kh == 7) || !(o.sh == 1 || o.sh == 2)) return false;
  if (o.inputs.size() > 8) return false;
  for (int u : o.inputs)
    if (g.ops[u].Cp != g.ops[o.inputs[0]].Cp) return false;
  // multi-input units (RandWire aggregation) have no halo path: their register-window form is
  // slower than the two-problem form, so they stay unfused unless IOS_FUSE_DW=2
  if (o.inputs.size() > 1 && !(getenv("IOS_FUSE_DW") && atoi(getenv("IOS_FUSE_DW")) >= 2)) return false;
  // halo path: one chunk's depthwise weights (k*k x 128 B of channels, held as fp32) in 8 KB
  if (o.inputs.size() == 1 && o.kh * o.kw * (kChunkBytes / g.esize()) * 4 > kHaloWBytes / 2) return false;
  if (o.inputs.size() == 1) {
    // measured (tools/op_report.py, NASNet-A / RandWire, 1 B200): fusion pays for 5x5/7x7 windows
    // and strided 3x3; a 3x3 stride-1 depthwise is cheap enough that the separate SIMT tile spread
    // over all SMs wins; windows whose 16 KB halo leaves patch tiles under 32 pixels (7x7 stride
    // 2) would launch hundreds of tiny tiles
    if (o.kh == 3 && o.sh == 1 && !(getenv("IOS_FUSE_DW") && atoi(getenv("IOS_FUSE_DW")) >= 3)) return false;
    const TTGeom tg = halo_geometry(g.batch, o.H, o.W, o.kh, o.sh, g.math == IOS_MATH_BF16 ? 2 : 4);
    if (tg.tR * tg.tWt < 32) return false;
  }
  return true;
}

// Halo-path patch tiles (single-input fused Relu-SepConv): the tile's input window
// ((tWt-1)s+k) x ((tR-1)s+k) pixels x 128 B must fit kHaloBytes, at most 32 quads (2 items per
// producer thread per chunk) and 128 pixels; most output pixels per tile, then fewest tiles.
TTGeom halo_geometry(int batch, int Ho, int Wo, int k, int s, int qw) {
  TTGeom best;
  int best_px = 0;
  for (int wt = std::min(Wo, kBM); wt >= 1; --wt) {
    const int ws = (wt - 1) * s + k;
    if (ws > 256) continue;
    const int qpr = (wt + qw - 1) / qw;
    for (int r = std::min(Ho, kBM / wt); r >= 1; --r) {
      const int hs = (r - 1) * s + k;
      if (hs > 256 || ws * hs * kChunkBytes > kHaloBytes / 2 || qpr * r > 32) continue;
      const int th = (Ho + r - 1) / r, tw = (Wo + wt - 1) / wt;
      const int tiles = batch * th * tw;
      const int px = r * wt;
      if (best.tiles == 0 || tiles < best.tiles || (tiles == best.tiles && px > best_px)) {
        best.tN = 1; best.tR = r; best.tWt = wt;
        best.tiles_h = th; best.tiles_w = tw; best.tiles = tiles;
        best_px = px;
      }
      break;   // the largest r that fits is best for this wt
    }
  }
  return best;
}

bool tap_tma_enabled() {
  static const bool on = [] {
    const char* v = getenv("IOS_TAP_TMA");
    return v ? atoi(v) != 0 : true;
  }();
  return on;
}

bool swap_enabled() {
  static const bool on = [] {
    const char* v = getenv("IOS_SWAP_AB");
    return v ? atoi(v) != 0 : true;
  }();
  return on;
}

// Tiling knobs (env overrides are for experiments; defaults from Inception V3 b=1 sweeps)
struct TileKnobs {
  int target_units;   // stop refining once the stage has this many units (0 = #SMs)
  int min_cps;        // never split K below this many 128 B chunks per unit
  int min_bn_small;   // narrowest N tile for small-M (<= 2 m-tiles) GEMMs
  int min_bn;         // narrowest N tile otherwise
  int one_wave;       // never refine past the target unit count (one wave of CTAs)
  int simt_in_target; // count SIMT tiles toward the target
  int max_split;      // most K splits per GEMM
};
static TileKnobs tile_knobs() {
  static TileKnobs k = [] {
    auto env = [](const char* n, int d) {
      const char* v = getenv(n);
      return v ? atoi(v) : d;
    };
    return TileKnobs{env("IOS_TARGET_UNITS", 0), env("IOS_MIN_CPS", 4), env("IOS_MIN_BN_SMALL", 16),
                     env("IOS_MIN_BN", 32), env("IOS_ONE_WAVE", 1), env("IOS_SIMT_IN_TARGET", 0),
                     env("IOS_MAX_SPLIT", 32)};
  }();
  return k;
}

// Tiling variants the stage tuner (ios_schedule_tune) may pick per stage: 0 = the default knobs,
// 1 = finer split-K (>= 2 chunks per unit), 2 = coarser split-K (>= 8 chunks per unit), 3 = cluster
// split-K (the default knobs on the cluster launch's co-resident grid, split counts rounded so the
// splits of a tile are summed in distributed shared memory: csplit 4 or 2). Measured: the best
// split-K granularity differs by network and stage (profiles/r1_kernel_ab_findings.md §5).
constexpr int kTileVariants = 4;
constexpr int kVariantCluster = 3;
// the DSMEM group size of a split count (cluster split-K variant)
int cluster_split_of(int split) { return split % 4 == 0 ? 4 : split % 2 == 0 ? 2 : 1; }
void choose_tiling(std::vector<GemmSpec*>& gs, int simt_tiles, int num_sms, int variant = 0) {
  TileKnobs kn = tile_knobs();
  if (variant == 1) kn.min_cps = std::max(1, kn.min_cps / 2);
  if (variant == 2) kn.min_cps = kn.min_cps * 2;
  const bool csk = variant == kVariantCluster;
  const int target = kn.target_units > 0 ? kn.target_units : num_sms;
  for (GemmSpec* p : gs) {
    if (p->swap) {
      // swap-AB: MMA M = 128 output channels (weight rows), MMA N = all pixels, one pixel tile
      p->BN = round_up(p->M, 16);
      p->ntn = 1;
      p->mt = (p->Npad8 + kBM - 1) / kBM;
      p->split = 1;
      p->cps = p->kch;
      continue;
    }
    p->mt = p->tt_tiles ? p->tt_tiles : (p->M + kBM - 1) / kBM;
    if (p->N16 <= p->max_bn) {
      p->BN = p->N16;
    } else {
      const int nt = (p->N16 + p->max_bn - 1) / p->max_bn;
      p->BN = round_up((p->N16 + nt - 1) / nt, 16);
    }
    p->ntn = (p->N16 + p->BN - 1) / p->BN;
    p->split = 1;
    p->cps = p->kch;
  }
  // Fill the SMs: refine the problem with the most expensive tile (N halving first, then split-K)
  // until there are about as many units as the target.
  for (int it = 0; it < 256; ++it) {
    // SIMT tiles mostly run in another phase (a depthwise before its pointwise GEMM, pools beside
    // short GEMMs), so by default the GEMM units alone are sized to one wave
    int units = kn.simt_in_target ? simt_tiles : 0;
    for (GemmSpec* p : gs) units += p->mt * p->ntn * p->split;
    if (units >= target) break;
    GemmSpec* best = nullptr;
    double best_cost = 0;
    for (GemmSpec* p : gs) {
      // small-M GEMMs are weight-bound: narrow N tiles first (A is small and L2-resident), then split K
      const int min_bn = p->mt <= 2 ? kn.min_bn_small : kn.min_bn;
      const int min_cps = p->fdw ? 1 : kn.min_cps;
      const bool can_n = !p->swap && !p->fdw && p->BN >= 2 * min_bn;
      // halo-path fused units pipeline their chunks in one CTA (no split-K finalize round)
      const bool can_k = p->cps >= 2 * min_cps && p->split < kn.max_split && p->fdw != 2;
      if (!can_n && !can_k) continue;
      const double c = p->cps * p->chunk_cost * (1.0 + p->BN / 256.0);
      if (c > best_cost) {
        best_cost = c;
        best = p;
      }
    }
    if (!best) break;
    // never refine past one wave: a step that would push the unit count over the target is
    // replaced by the largest split-K that still fits, or refinement stops
    const int cur = best->mt * best->ntn * best->split;
    const int others = units - cur;
    const bool can_n = !best->swap && !best->fdw && best->BN >= 2 * (best->mt <= 2 ? kn.min_bn_small : kn.min_bn);
    const int best_min_cps = best->fdw ? 1 : kn.min_cps;
    if (can_n && (!kn.one_wave || others + 2 * cur <= target)) {
      best->BN = round_up(best->BN / 2, 16);
      best->ntn = (best->N16 + best->BN - 1) / best->BN;
    } else {
      int want = std::min(best->split * 2, kn.max_split);
      const int room = (target - others) / (best->mt * best->ntn);
      if (kn.one_wave && want > room) want = room;
      if (csk && want > 2) want = want >= 4 ? want / 4 * 4 : 2;   // splits a DSMEM group can sum
      if (want <= best->split || (best->kch + want - 1) / want < best_min_cps) break;
      best->cps = (best->kch + want - 1) / want;
      best->split = (best->kch + best->cps - 1) / best->cps;
    }
  }
}

struct PlanBuilder {
  Graph& g;
  DeviceState& d;
  std::vector<Problem> probs;
  std::vector<View> views;
  std::vector<Segment> segs;
  std::vector<GemmSpec> specs;       // parallel to probs (GEMM problems only meaningful)
  std::map<int, std::vector<int>> op_probs;  // op -> its problems (last one produces the output)

  explicit PlanBuilder(Graph& gg) : g(gg), d(*gg.dev) {}

  int add_problem(int kind) {
    Problem p{};
    p.kind = kind;
    p.dtype = g.dtype();
    p.split = 1;
    probs.push_back(p);
    specs.push_back(GemmSpec{});
    return (int)probs.size() - 1;
  }
  // completion counters of the in-stage producers of op u's output (through elided ops)
  void producers(int u, const std::vector<int>& stage_ops, std::vector<int>& out) {
    if (u == 0 || !std::binary_search(stage_ops.begin(), stage_ops.end(), u)) return;
    auto it = op_probs.find(u);
    if (it != op_probs.end() && !it->second.empty()) {
      out.push_back(it->second.back());
      return;
    }
    for (int w : g.ops[u].inputs) producers(w, stage_ops, out);   // elided concat / identity
  }
  void add_deps(int pi, const std::vector<int>& deps) {
    Problem& p = probs[pi];
    for (int q : deps) {
      bool dup = false;
      for (int k = 0; k < p.n_deps; ++k) dup |= p.dep_idx[k] == q;
      if (dup) continue;
      if (p.n_deps >= 6) IOS_FAIL(IOS_ERR_UNSUPPORTED, "stage member with more than 6 in-stage producers");
      p.dep_idx[p.n_deps++] = q;   // problem index for now; turned into counter index later
    }
  }
  int gemm(int in_op_view_src, const View& in, void* wpack, int n8, float* bias, int Ntot, int kh, int kw, int sh,
           int sw, int ph, int pw, int Ho, int Wo, int flags, int kblk = 0) {
    (void)in_op_view_src;
    const int pi = add_problem(PK_GEMM);
    Problem& p = probs[pi];
    p.batch = g.batch;
    p.flags = flags;
    p.kh = kh; p.kw = kw; p.sh = sh; p.sw = sw; p.ph = ph; p.pw = pw;
    p.Ho = Ho; p.Wo = Wo;
    p.in_begin = (int)views.size();
    p.n_in = 1;
    views.push_back(in);
    p.wts = (uint64_t)wpack;
    p.Npad8 = n8;
    p.bias = (uint64_t)bias;
    p.M = g.batch * Ho * Wo;
    const int elems = kChunkBytes / g.esize();
    p.K = kblk ? kh * kw * kblk * elems : kh * kw * in.C;
    p.k_chunks = (p.K + elems - 1) / elems;
    p.seg_begin = (int)segs.size();
    GemmSpec& s = specs[pi];
    s.Npad8 = n8;
    s.swap = (p.M <= kBM && swap_enabled() && g.math != IOS_MATH_FP32_SIMT) ? 1 : 0;
    if (kblk) {
      const TTGeom tg = tt_geometry(g.batch, Ho, Wo, sh, sw);
      p.tt = 1;
      p.kblk = kblk;
      p.tN = tg.tN; p.tR = tg.tR; p.tWt = tg.tWt;
      p.tiles_h = tg.tiles_h; p.tiles_w = tg.tiles_w;
      s.tt_tiles = tg.tiles;
      if (tg.tiles != 1) s.swap = 0;   // swap-AB needs the whole image as one dense pixel tile
    }
    s.max_bn = g.math == IOS_MATH_FP32_SIMT ? 32 : kMaxBN;   // SIMT: 32 columns in registers
    s.M = p.M;
    s.N16 = round_up(Ntot, 16);
    s.K = p.K;
    s.kch = p.k_chunks;
    return pi;
  }
  void seg(int pi, int n0, int n1, const View& out, int relu) {
    Segment s{};
    s.n0 = n0;
    s.n1 = n1;
    s.out = out;
    s.relu = relu;
    segs.push_back(s);
    probs[pi].n_seg++;
  }
  int simt(int kind, const Op& o, const std::vector<int>& inputs, const View& out, int flags) {
    const int pi = add_problem(kind);
    Problem& p = probs[pi];
    p.batch = g.batch;
    p.flags = flags;
    p.kh = o.kh; p.kw = o.kw; p.sh = o.sh; p.sw = o.sw; p.ph = o.ph; p.pw = o.pw;
    p.Ho = o.H; p.Wo = o.W;
    p.in_begin = (int)views.size();
    p.n_in = (int)inputs.size();
    for (int u : inputs) views.push_back(d.od[u].out);
    p.out = out;
    return pi;
  }
};

// The driver's tensor-map encoder, resolved through the runtime (no link-time libcuda dependency:
// the library must load on machines without a driver).
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<EncodeTiledFn>(f);
  }();
  if (!fn) IOS_FAIL(IOS_ERR_CUDA, "cuTensorMapEncodeTiled is unavailable");
  return fn;
}

void free_plan(DeviceState& d, StagePlan* p) {
  if (!p) return;
  for (void* a : p->allocs) cudaFreeAsync(a, d.stream);
  delete p;
}

StagePlan* build_plan(Graph& g, int bpos, uint64_t mask, int strategy, int variant = -1) {
  DeviceState& d = *g.dev;
  if (variant < 0) {
    // untuned stages: the default knobs, or IOS_TILE_VARIANT (experiments / tests of one variant)
    auto vit = d.tile_variant.find(std::make_tuple(bpos, mask, strategy));
    const char* ev = getenv("IOS_TILE_VARIANT");
    const int dv = ev ? std::max(0, std::min(kTileVariants - 1, atoi(ev))) : 0;
    variant = vit == d.tile_variant.end() ? dv : vit->second;
  }
  const std::vector<int> ops = g.ops_of(bpos, mask);
  PlanBuilder b(g);
  auto* plan = new StagePlan();
  // cluster split-K variant: tiles sized for the cluster launch's co-resident grid (GPC sizes leave
  // fewer SMs than the plain one-CTA-per-SM grid); no cluster support -> the default tiling
  if (variant == kVariantCluster && (d.cluster_ctas <= 0 || g.math == IOS_MATH_FP32_SIMT)) variant = 0;
  const int grid_sms = variant == kVariantCluster ? d.cluster_ctas : d.num_sms;
  try {
    if (strategy == IOS_MERGE) {
      // ---- operator merge (Z4): bounding-box kernel, stacked zero-padded filters,
      // one GEMM; the split is the epilogue writing each branch's channel slice.
      if (!g.mergeable(ops)) IOS_FAIL(IOS_ERR_NOT_MERGEABLE, "stage is not mergeable");
      int st_h = 1 << 30, en_h = -(1 << 30), st_w = 1 << 30, en_w = -(1 << 30);
      for (int v : ops) {
        const Op& o = g.ops[v];
        st_h = std::min(st_h, -o.ph); en_h = std::max(en_h, -o.ph + o.kh);
        st_w = std::min(st_w, -o.pw); en_w = std::max(en_w, -o.pw + o.kw);
      }
      const int KH = en_h - st_h, KW = en_w - st_w, PH = -st_h, PW = -st_w;
      const Op& f = g.ops[ops[0]];
      const Op& x = g.ops[f.inputs[0]];
      std::vector<int> row0;
      int ntot = 0;
      for (int v : ops) {
        row0.push_back(ntot);
        ntot += g.ops[v].Cp;
      }
      const int cin = x.C, cin_p = x.Cp;
      const int kblk = tap_tma_blocks(g, cin_p, KH, KW, f.sh, f.sw, PH, PW, f.flags, g.batch, f.H, f.W);
      const int tapk = kblk ? kblk * (kChunkBytes / g.esize()) : cin_p;
      int merged_n8 = 0;
      plan->merged_pack = pack_gemm(d, ntot, KH * KW * tapk, g.dtype(), [&](int nn, int k) -> float {
        int bi = (int)ops.size() - 1;
        while (row0[bi] > nn) --bi;
        const Op& o = g.ops[ops[bi]];
        const int r = nn - row0[bi];
        if (r >= o.cout) return 0.0f;
        const int tap = k / tapk, ci = k % tapk;
        if (ci >= cin) return 0.0f;
        const int i = tap / KW - (-o.ph - st_h), j = tap % KW - (-o.pw - st_w);
        if (i < 0 || i >= o.kh || j < 0 || j >= o.kw) return 0.0f;
        return o.weight[(((size_t)r * cin + ci) * o.kh + i) * o.kw + j];
      }, &merged_n8, &plan->allocs);
      std::vector<float> bias((size_t)round_up(ntot, 256) + 16, 0.0f);
      for (size_t bi = 0; bi < ops.size(); ++bi) {
        const Op& o = g.ops[ops[bi]];
        for (int c = 0; c < o.cout; ++c) bias[row0[bi] + c] = o.bias[c];
      }
      plan->merged_bias = upload(d, bias, 0, &plan->allocs);
      const int pi = b.gemm(f.inputs[0], d.od[f.inputs[0]].out, plan->merged_pack, merged_n8, plan->merged_bias,
                            ntot, KH, KW, f.sh, f.sw, PH, PW, f.H, f.W, f.flags & IOS_F_RELU_PRE, kblk);
      for (size_t bi = 0; bi < ops.size(); ++bi) {
        const Op& o = g.ops[ops[bi]];
        b.seg(pi, row0[bi], row0[bi] + o.Cp, d.od[ops[bi]].out, (o.flags & IOS_F_RELU_POST) ? 1 : 0);
      }
      for (int v : ops) b.op_probs[v] = {pi};
    } else {
      // ---- concurrent execution: every member op in one launch; groups emerge from dependencies
      for (int v : ops) {
        const Op& o = g.ops[v];
        OpDev& e = d.od[v];
        std::vector<int> deps;
        for (int u : o.inputs) b.producers(u, ops, deps);
        switch (o.kind) {
          case IOS_OP_CONV:
          case IOS_OP_LINEAR: {
            const int u = o.inputs[0];
            const int pi = e.unfold ? b.gemm(u, d.unfold_view, e.wpack, e.wpack_n8, e.bias, o.Cp, o.kh, 1, o.sh, 1, o.ph, 0,
                                             o.H, o.W, 0, 1)
                                    : b.gemm(u, d.od[u].out, e.wpack, e.wpack_n8, e.bias, o.Cp, o.kh, o.kw, o.sh, o.sw, o.ph,
                                             o.pw, o.H, o.W, o.flags & IOS_F_RELU_PRE, e.kblk);
            b.seg(pi, 0, o.Cp, e.out, (o.flags & IOS_F_RELU_POST) ? 1 : 0);
            b.add_deps(pi, deps);
            b.op_probs[v] = {pi};
            break;
          }
          case IOS_OP_SEPCONV: {
            if (fuse_dw_ok(g, o)) {
              // fused Relu-SepConv: ONE GEMM problem whose producer computes the
              // depthwise half into the A operand; M tiles are output patches (epilogue mapping of
              // tap-TMA tiles), K = the input channels
              const int u0 = o.inputs[0];
              const int pi = b.gemm(-1, d.od[u0].out, e.wpack, e.wpack_n8, e.bias, o.Cp, 1, 1, 1, 1, 0, 0, o.H, o.W, 0);
              for (size_t k = 1; k < o.inputs.size(); ++k) b.views.push_back(d.od[o.inputs[k]].out);
              Problem& p = b.probs[pi];
              p.n_in = (int)o.inputs.size();
              p.fdw = 1;
              p.dk = o.kh; p.ds = o.sh; p.dp = o.ph;
              p.dH = g.ops[u0].H; p.dW = g.ops[u0].W;
              p.dww = (uint64_t)e.dw;
              p.add_w = (uint64_t)e.add_w;
              const int qw = g.math == IOS_MATH_BF16 ? 2 : 4;
              const bool halo = o.inputs.size() == 1;   // fuse_dw_ok admits multi-input units only with IOS_FUSE_DW=2
              const TTGeom tg = halo ? halo_geometry(g.batch, o.H, o.W, o.kh, o.sh, qw) : fdw_geometry(g.batch, o.H, o.W, qw);
              if (halo) {
                p.hws = (tg.tWt - 1) * o.sw + o.kw;
                p.hhs = (tg.tR - 1) * o.sh + o.kh;
                p.dwc = (uint64_t)e.dwc;
              }
              p.tt = 1;
              p.tN = tg.tN; p.tR = tg.tR; p.tWt = tg.tWt;
              p.tiles_h = tg.tiles_h; p.tiles_w = tg.tiles_w;
              GemmSpec& sp = b.specs[pi];
              sp.tt_tiles = tg.tiles;
              sp.swap = 0;
              sp.fdw = halo ? 2 : 1;
              sp.chunk_cost = 1.0 + o.kh * o.kw / 4.0;
              b.seg(pi, 0, o.Cp, e.out, (o.flags & IOS_F_RELU_POST) ? 1 : 0);
              b.add_deps(pi, deps);
              b.op_probs[v] = {pi};
              break;
            }
            Op dwop = o;
            const int pd = b.simt(PK_DWCONV, dwop, o.inputs, e.dw_out, o.flags);
            b.probs[pd].wts = (uint64_t)e.dw;
            b.probs[pd].add_w = (uint64_t)e.add_w;
            b.add_deps(pd, deps);
            const int pi = b.gemm(-1, e.dw_out, e.wpack, e.wpack_n8, e.bias, o.Cp, 1, 1, 1, 1, 0, 0, o.H, o.W, 0);
            b.seg(pi, 0, o.Cp, e.out, (o.flags & IOS_F_RELU_POST) ? 1 : 0);
            b.add_deps(pi, {pd});
            b.op_probs[v] = {pd, pi};
            break;
          }
          case IOS_OP_MAXPOOL:
          case IOS_OP_AVGPOOL:
          case IOS_OP_GLOBAL_AVGPOOL:
          case IOS_OP_ADD: {
            const int kind = o.kind == IOS_OP_MAXPOOL ? PK_MAXPOOL
                             : o.kind == IOS_OP_AVGPOOL ? PK_AVGPOOL
                             : o.kind == IOS_OP_ADD ? PK_ADD : PK_GAVGPOOL;
            const int pi = b.simt(kind, o, o.inputs, e.out, o.flags);
            b.probs[pi].add_w = (uint64_t)e.add_w;
            b.add_deps(pi, deps);
            b.op_probs[v] = {pi};
            break;
          }
          case IOS_OP_CONCAT:
          case IOS_OP_IDENTITY: {
            if (e.elided) break;   // realised by addressing: no work, completion = its producers'
            const int pi = b.simt(PK_COPY, o, o.inputs, e.out, o.flags);
            b.add_deps(pi, deps);
            b.op_probs[v] = {pi};
            break;
          }
          default:
            IOS_FAIL(IOS_ERR_UNSUPPORTED, "op kind");
        }
      }
    }
    // ---- tiling
    const int nv = 16 / g.esize();
    int simt_tiles = 0;
    for (size_t i = 0; i < b.probs.size(); ++i) {
      Problem& p = b.probs[i];
      if (p.kind == PK_GEMM) continue;
      const int nvec = p.out.C / nv;
      const bool sq = p.kh == p.kw && p.sh == p.sw && (p.sh == 1 || p.sh == 2);
      const bool win = sq && ((p.kind == PK_DWCONV && (p.kh == 3 || p.kh == 5 || p.kh == 7) && p.n_in <= 8) ||
                              ((p.kind == PK_MAXPOOL || p.kind == PK_AVGPOOL) && p.kh == 3));
      if (p.kind == PK_GAVGPOOL) {
        // 4 items per warp that runs SIMT tiles: the 4 epilogue warps, or all 9 warps of a stage
        // without GEMM members (more loads in flight per SM at large batch)
        bool any_gemm = false;
        for (const Problem& q : b.probs) any_gemm |= q.kind == PK_GEMM;
        p.n_items = p.batch * nvec;
        p.items_per_tile = any_gemm ? 16 : 4 * (kThreads / 32);
      } else if (win) {
        // quads of horizontally adjacent outputs (win_tile in stage_kernel.cu); one quad x vector
        // per thread of a 128-thread tile
        p.dwq = g.esize() == 2 ? 2 : 4;
        p.n_items = p.batch * p.Ho * ((p.Wo + p.dwq - 1) / p.dwq);
        p.items_per_tile = std::max(1, 128 / std::max(1, nvec));
      } else {
        // about 2 vector items per epilogue thread so the stage spreads over many SMs
        p.n_items = p.batch * p.Ho * p.Wo;
        p.items_per_tile = std::max(1, 256 / std::max(1, nvec));
      }
      // never more tiles than CTAs for one problem: a second wave doubles a latency-bound op
      if (p.kind != PK_GAVGPOOL)
        p.items_per_tile = std::max(p.items_per_tile, (p.n_items + grid_sms - 1) / grid_sms);
      p.n_tiles = (p.n_items + p.items_per_tile - 1) / p.items_per_tile;
      simt_tiles += p.n_tiles;
    }
    // Phase-aware tiling: members of one intra-group chain never run at the same time (a member
    // waits for its producer's completion counter), so each dependency phase (0 = no in-stage
    // producer, k = 1 + the latest producer's phase) is sized to fill the SMs on its own, instead of
    // all members sharing one wave (measured on Inception Mixed_5b: the 5x5 and 3x3 links of the
    // chains got 20-40 CTAs with 14-27 K chunks each).
    // (opt-in, IOS_PHASE_TILING=1: measured 2 % slower on the Inception V3 IOS schedule -- the extra
    // split-K reductions of the first links cost more than the shorter K loops of the later ones)
    static const bool phased = getenv("IOS_PHASE_TILING") && atoi(getenv("IOS_PHASE_TILING")) != 0;
    std::vector<int> phase(b.probs.size(), 0);
    int n_phases = 1;
    for (size_t i = 0; i < b.probs.size(); ++i) {
      for (int k = 0; k < b.probs[i].n_deps; ++k)   // dep_idx still holds problem indices here
        phase[i] = std::max(phase[i], phase[b.probs[i].dep_idx[k]] + 1);
      n_phases = std::max(n_phases, phase[i] + 1);
    }
    if (!phased) std::fill(phase.begin(), phase.end(), 0), n_phases = 1;
    for (int ph = 0; ph < n_phases; ++ph) {
      std::vector<GemmSpec*> gs;
      int ph_simt = 0;
      for (size_t i = 0; i < b.probs.size(); ++i) {
        if (phase[i] != ph) continue;
        if (b.probs[i].kind == PK_GEMM) gs.push_back(&b.specs[i]);
        else ph_simt += b.probs[i].n_tiles;
      }
      if (!gs.empty()) choose_tiling(gs, phased ? ph_simt : simt_tiles, grid_sms, variant);
    }
    size_t ws_bytes = 0;
    int n_tilectr = 0;
    for (size_t i = 0; i < b.probs.size(); ++i) {
      Problem& p = b.probs[i];
      if (p.kind != PK_GEMM) continue;
      const GemmSpec& s = b.specs[i];
      const View& in = b.views[p.in_begin];
      p.fd_howo = make_fastdiv((uint32_t)(p.Ho * p.Wo));
      p.fd_wo = make_fastdiv((uint32_t)p.Wo);
      p.fd_split = make_fastdiv((uint32_t)s.split);
      p.fd_q4 = make_fastdiv((uint32_t)std::max(1, s.BN / 4));
      p.fd_ntn = make_fastdiv((uint32_t)s.ntn);
      p.fd_cin = make_fastdiv((uint32_t)in.C);
      p.fd_kw = make_fastdiv((uint32_t)p.kw);
      if (p.tt) {
        p.fd_kblk = make_fastdiv((uint32_t)std::max(1, p.kblk));
        p.fd_thw = make_fastdiv((uint32_t)(p.tR * p.tWt));
        p.fd_tw = make_fastdiv((uint32_t)p.tWt);
        p.fd_tilw = make_fastdiv((uint32_t)p.tiles_w);
        p.fd_tilh = make_fastdiv((uint32_t)p.tiles_h);
      }
      // A via TMA when it is a plain [M, C] matrix: 1x1, stride 1, no padding, no pre-ReLU
      p.a_tma = (g.math != IOS_MATH_FP32_SIMT && !p.fdw && p.kh == 1 && p.kw == 1 && p.sh == 1 && p.sw == 1 && p.ph == 0 && p.pw == 0 &&
                 !(p.flags & IOS_F_RELU_PRE)) ? 1 : 0;
      p.swap_ab = s.swap;
      p.BN = s.BN;
      p.n_tiles_n = s.ntn;
      p.m_tiles = s.mt;
      p.split = s.split;
      p.chunks_per_split = s.cps;
      p.n_tiles = s.mt * s.ntn * s.split;
      p.csplit = 1;
      if (p.split > 1) {
        p.workspace = ws_bytes;   // offset for now
        // one fp32 partial slab per split (<= kSlabSplits), else one zeroed reduction slab
        static const int slab_splits = getenv("IOS_SLAB_SPLITS") ? atoi(getenv("IOS_SLAB_SPLITS")) : kSlabSplits;
        p.slabs = s.split <= slab_splits ? 1 : 0;
        const size_t copies = p.slabs ? s.split : 1;
        ws_bytes += (size_t)s.mt * s.ntn * copies * kBM * s.BN * sizeof(float);
        p.tilectr_idx = n_tilectr;
        n_tilectr += s.mt * s.ntn;
      }
    }
    // ---- cluster split-K (variant 3): the csplit splits of an output tile are consecutive tiles
    // starting at a multiple of csplit, so with a grid that is a multiple of the cluster size they
    // run at the same time on consecutive ranks of one cluster (a halo-path stage keeps its fixed
    // ring: no receive buffer; per-split slabs keep the deterministic global path)
    bool csk_plan = false;
    if (variant == kVariantCluster) {
      bool halo = false;
      for (Problem& p : b.probs) halo |= p.kind == PK_GEMM && p.hws != 0;
      for (Problem& p : b.probs) {
        if (p.kind != PK_GEMM || p.split < 2 || p.swap_ab || p.slabs || halo) continue;
        p.csplit = cluster_split_of(p.split);
        csk_plan |= p.csplit > 1;
      }
    }
    for (Problem& p : b.probs)
      if (p.kind != PK_GEMM) p.csplit = 1;
    // ---- tiles and counters: problems keep insertion (topological) order, so deps point back
    const int np = (int)b.probs.size();
    if (np > kMaxProblems) IOS_FAIL(IOS_ERR_UNSUPPORTED, "too many problems in one stage");
    int tiles = 0;
    for (Problem& p : b.probs) {
      // padding tiles (skipped by every role) keep a csplit group on one cluster
      if (csk_plan && p.csplit > 1) tiles = round_up(tiles, kClusterCtas);
      p.tile_begin = tiles;
      tiles += p.n_tiles;
    }
    // ---- row-band dependencies: a consumer tile waits only for the producer tiles
    // covering the input rows it reads, when both sides' tiles map to output rows (not swap-AB, not
    // a global pool) and the producer's output is the consumer's input grid (IOS_ROW_BANDS=0: off)
#ifdef IOS_ROW_BANDS
    static const bool row_bands = !getenv("IOS_ROW_BANDS") || atoi(getenv("IOS_ROW_BANDS")) != 0;
#else
    constexpr bool row_bands = false;   // opt-in build (stage_kernel.cu: measured net loss by default)
#endif
    std::vector<DepBand> bands;
    std::vector<int> band_n(np, 0);   // bands of producer q that some consumer waits on (0: none)
    for (int i = 0; i < np; ++i) {
      Problem& p = b.probs[i];
      p.band_begin = -1;
      p.band_ctr = -1;
      if (!row_bands || p.n_deps == 0) continue;
      const bool rows_ok = !(p.kind == PK_GEMM && p.swap_ab) && p.kind != PK_GAVGPOOL;
      const View& in = b.views[p.in_begin];
      p.band_begin = (int)bands.size();
      for (int k = 0; k < p.n_deps; ++k) {
        const int qi = p.dep_idx[k];
        const Problem& q = b.probs[qi];
        DepBand db{};
        db.H = q.Ho;
        db.W = q.Wo;
        if (rows_ok && q.Ho == in.H && q.Wo == in.W && q.batch == p.batch) {
          if (q.kind == PK_GEMM && !q.swap_ab) {
            db.mode = q.tt ? 2 : 1;
            db.bsz = kBM;
            db.tN = q.tN;
            db.tR = q.tR;
            db.tiles_h = q.tiles_h;
            db.tiles_w = q.tiles_w;
            db.target = q.n_tiles_n * q.split;
            db.nbands = q.m_tiles;
          } else if (q.kind != PK_GEMM && q.kind != PK_GAVGPOOL) {
            db.mode = q.dwq ? 4 : 3;
            db.bsz = q.items_per_tile;
            db.tiles_w = q.dwq ? (q.Wo + q.dwq - 1) / q.dwq : 0;
            db.target = 1;
            db.nbands = q.n_tiles;
          }
        }
        if (db.mode) band_n[qi] = db.nbands;
        bands.push_back(db);
      }
    }
    int n_counters = kCounterBase + np + n_tilectr;
    for (int i = 0; i < np; ++i)
      if (band_n[i]) {
        b.probs[i].band_ctr = n_counters;
        n_counters += band_n[i];
      }
    for (int i = 0; i < np; ++i) {
      Problem& p = b.probs[i];
      p.done_idx = kCounterBase + i;
      for (int k = 0; k < p.n_deps; ++k) {
        const Problem& q = b.probs[p.dep_idx[k]];
        if (p.band_begin >= 0 && bands[p.band_begin + k].mode) bands[p.band_begin + k].ctr = q.band_ctr;
        p.dep_target[k] = q.n_tiles;   // every unit (incl. each split-K part) signals once
        p.dep_idx[k] = kCounterBase + p.dep_idx[k];
      }
      if (p.kind == PK_GEMM && p.split > 1) p.tilectr_idx += kCounterBase + np;
    }
    plan->empty = tiles == 0;
    if (!plan->empty) {
      if (ws_bytes) plan->workspace = dmalloc(d, ws_bytes, &plan->allocs);
      for (Problem& p : b.probs)
        if (p.kind == PK_GEMM && p.split > 1) p.workspace += (uint64_t)plan->workspace;
      const size_t pb = b.probs.size() * sizeof(Problem), vb = b.views.size() * sizeof(View),
                   sb = b.segs.size() * sizeof(Segment), bb = bands.size() * sizeof(DepBand);
      // a problem signals completion only if a later member of the stage waits on it
      for (Problem& p : b.probs)
        for (int k = 0; k < p.n_deps; ++k) b.probs[p.dep_idx[k] - kCounterBase].signal = 1;
      std::vector<uint8_t> blob(pb + vb + sb + bb + 64, 0);
      std::memcpy(blob.data(), b.probs.data(), pb);
      if (vb) std::memcpy(blob.data() + pb, b.views.data(), vb);
      if (sb) std::memcpy(blob.data() + pb + vb, b.segs.data(), sb);
      if (bb) std::memcpy(blob.data() + pb + vb + sb, bands.data(), bb);
      // tensor maps for TMA-loaded A operands (global memory, 64 B aligned, written before launch)
      std::vector<CUtensorMap> maps;
      const CUtensorMapDataType tdt =
          g.math == IOS_MATH_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
      const cuuint32_t elems = (cuuint32_t)(kChunkBytes / g.esize());
      for (Problem& p : b.probs) {
        if (p.kind != PK_GEMM || (p.fdw && !p.hws) || !(p.a_tma || p.tt)) continue;
        const View& in = b.views[p.in_begin];
        CUtensorMap tm;
        void* base = reinterpret_cast<char*>(in.ptr) + (size_t)in.coff * g.esize();
        CUresult r;
        if (p.hws) {
          // fused Relu-SepConv halo: NHWC input {C, W, H, N}, box = one 128 B channel chunk of an
          // hhs x hws input window, dense (no swizzle); padding = out-of-bounds zeros
          const cuuint64_t dims[4] = {(cuuint64_t)in.C, (cuuint64_t)in.W, (cuuint64_t)in.H, (cuuint64_t)p.batch};
          const cuuint64_t rs = (cuuint64_t)in.cstride * g.esize();
          const cuuint64_t strides[3] = {rs, rs * in.W, rs * in.W * in.H};
          const cuuint32_t box[4] = {elems, (cuuint32_t)p.hws, (cuuint32_t)p.hhs, 1};
          const cuuint32_t estr[4] = {1, 1, 1, 1};
          r = encode_tiled()(&tm, tdt, 4, base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                             CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
          if (r != CUDA_SUCCESS) IOS_FAIL(IOS_ERR_CUDA, "halo tensor map rejected by the driver");
        } else if (p.a_tma) {
          // [M, C] matrix: 128 rows x 128 B per box
          const cuuint64_t dims[2] = {(cuuint64_t)in.C, (cuuint64_t)p.M};
          const cuuint64_t strides[1] = {(cuuint64_t)in.cstride * g.esize()};
          const cuuint32_t box[2] = {elems, (cuuint32_t)kBM};
          const cuuint32_t estr[2] = {1, 1};
          r = encode_tiled()(&tm, tdt, 2, base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                             CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        } else {
          // NHWC input as a 4D tensor {C, W, H, N}; one box = tN x tR x tWt output pixels of one tap
          // (element strides = conv strides) x one 128 B channel block; padding = out-of-bounds zeros
          const cuuint64_t dims[4] = {(cuuint64_t)in.C, (cuuint64_t)in.W, (cuuint64_t)in.H, (cuuint64_t)p.batch};
          const cuuint64_t rs = (cuuint64_t)in.cstride * g.esize();
          const cuuint64_t strides[3] = {rs, rs * in.W, rs * in.W * in.H};
          const cuuint32_t box[4] = {elems, (cuuint32_t)(p.tWt * p.sw), (cuuint32_t)(p.tR * p.sh), (cuuint32_t)p.tN};
          const cuuint32_t estr[4] = {1, (cuuint32_t)p.sw, (cuuint32_t)p.sh, 1};
          r = encode_tiled()(&tm, tdt, 4, base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                             CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
          if (r != CUDA_SUCCESS) IOS_FAIL(IOS_ERR_CUDA, "tap-TMA tensor map rejected by the driver");
        }
        if (r != CUDA_SUCCESS) {
          p.a_tma = 0;   // fall back to the cp.async gather
          continue;
        }
        p.tmap_a = maps.size();
        maps.push_back(tm);
      }
      if (!maps.empty()) {
        void* mp = upload(d, maps, 0, &plan->allocs);
        for (Problem& p : b.probs)
          if (p.kind == PK_GEMM && (!p.fdw || p.hws) && (p.a_tma || p.tt)) p.tmap_a = (uint64_t)mp + p.tmap_a * sizeof(CUtensorMap);
      }
      std::memcpy(blob.data(), b.probs.data(), pb);
      plan->dmem = upload(d, blob, 0, &plan->allocs);
      plan->counters = static_cast<int*>(dmalloc(d, (size_t)n_counters * sizeof(int), &plan->allocs));
      StageDesc& sd = plan->sd;
      sd.problems = (uint64_t)plan->dmem;
      sd.views = (uint64_t)plan->dmem + pb;
      sd.segs = (uint64_t)plan->dmem + pb + vb;
      sd.counters = (uint64_t)plan->counters;
      sd.err = (uint64_t)d.err;
      sd.n_problems = np;
      sd.n_tiles = tiles;
      sd.n_counters = n_counters;
      sd.blob_bytes = (int)(pb + vb + sb + bb);
      sd.views_off = (int)pb;
      sd.segs_off = (int)(pb + vb);
      sd.bands_off = (int)(pb + vb + sb);
      sd.uses_counters = 0;
      for (Problem& p : b.probs) sd.uses_counters |= (p.signal || (p.kind == PK_GEMM && p.split > 1)) ? 1 : 0;
      sd.feat = 0;   // kernel feature class (stage_desc.h): which producer paths the stage uses
      for (Problem& p : b.probs) {
        if (p.kind != PK_GEMM) continue;
        if (p.fdw) sd.feat |= F_FDW;
        else if (!(p.a_tma || p.tt)) sd.feat |= F_GATHER;
      }
      // ring: slots sized for the stage's widest B operand (weights BN x 128 B, or the swap-AB pixel
      // operand), as many as fit kRingBytes: a 128 x 32 tile ring is 9 deep instead of 4. A stage
      // with a halo-path fused sepconv keeps the fixed 3 x 48 KB ring (the 4th slot holds its windows).
      int max_bn = 16;
      bool halo = false;
      for (Problem& p : b.probs) {
        if (p.kind != PK_GEMM) continue;
        // (a swap-AB plain-TMA tile's pixel box is always 128 rows, whatever its BN)
        max_bn = std::max(max_bn, (p.swap_ab && p.a_tma) ? kBM : p.BN);
        halo |= p.hws != 0;
      }
      static const int deep = getenv("IOS_DEEP_RING") ? atoi(getenv("IOS_DEEP_RING")) : 1;
      // cluster split-K receive buffer at the end of the ring region: (csplit - 1) peers x the owned
      // 128 / csplit rows x (BN fp32 + 16 B: conflict-free row-per-lane reads)
      // (one row stride for the stage: the widest csplit problem's; the largest group form is
      // csplit 4: 3 peers x 32 rows)
      int rstride = 0;
      for (Problem& p : b.probs)
        if (p.kind == PK_GEMM && p.csplit > 1) rstride = std::max(rstride, p.BN * 4 + 16);
      const int rbuf = rstride ? round_up((kBM - kBM / kClusterCtas) * rstride, 1024) : 0;
      if (halo || !deep) {
        sd.slot_bytes = kAStageBytes + kBStageBytes;
        sd.ring_slots = halo ? kStages - 1 : kStages;
      } else {
        sd.slot_bytes = kAStageBytes + round_up(max_bn * kChunkBytes, 1024);
        sd.ring_slots = std::min(kMaxSlots, (kRingBytes - rbuf) / sd.slot_bytes);
      }
      if (rbuf && (halo || sd.ring_slots < 2)) IOS_FAIL(IOS_ERR_UNSUPPORTED, "cluster split-K receive buffer does not fit");
      sd.cluster = csk_plan ? kClusterCtas : 1;
      sd.rbuf_off = kRingBytes - rbuf;
      sd.rbuf_stride = rstride;
      if (csk_plan) sd.feat |= F_CSK;
      sd.has_gemm = 0;
      for (Problem& p : b.probs) sd.has_gemm |= p.kind == PK_GEMM;
      plan->grid = std::min(tiles, d.num_sms);
      if (csk_plan) plan->grid = std::min(round_up(tiles, kClusterCtas), d.cluster_ctas);
      plan->dtype = g.dtype();
      const bool dump = getenv("IOS_DUMP_PLANS") && atoi(getenv("IOS_DUMP_PLANS")) != 0;
      if (dump) {   // diagnostics: one line per problem of every plan built
        fprintf(stderr, "[plan] block %d mask %llx T %d variant %d: %d tiles, grid %d, cluster %d, %d slots x %d B, feat %d\n",
                bpos, (unsigned long long)mask, strategy, variant, tiles, plan->grid, sd.cluster, sd.ring_slots,
                sd.slot_bytes, sd.feat);
        for (size_t i = 0; i < b.probs.size(); ++i) {
          const Problem& p = b.probs[i];
          if (p.kind == PK_GEMM)
            fprintf(stderr, "[plan]   gemm M %d N %d K %d kch %d | BN %d ntn %d mt %d split %d cps %d csplit %d | swap %d tma %d tt %d fdw %d deps %d\n",
                    p.M, b.specs[i].N16, p.K, p.k_chunks, p.BN, p.n_tiles_n, p.m_tiles, p.split, p.chunks_per_split,
                    p.csplit, p.swap_ab, p.a_tma, p.tt, p.fdw, p.n_deps);
          else
            fprintf(stderr, "[plan]   simt kind %d tiles %d items %d deps %d\n", p.kind, p.n_tiles, p.n_items, p.n_deps);
        }
      }
    }
  } catch (...) {
    free_plan(d, plan);
    throw;
  }
  return plan;
}

StagePlan* get_plan(Graph& g, int bpos, uint64_t mask, int strategy) {
  DeviceState& d = *g.dev;
  auto key = std::make_tuple(bpos, mask, strategy);
  auto it = d.plans.find(key);
  if (it != d.plans.end()) return it->second;
  StagePlan* p = build_plan(g, bpos, mask, strategy);
  d.plans[key] = p;
  return p;
}

void launch_plan(const StagePlan* p, cudaStream_t st) {
  if (p->empty) return;
  IOS_CHECK_CUDA(launch_stage(p->sd, p->dtype, p->grid, st));
}

}  // namespace

// The kernel's error flag lives in host-mapped pinned memory: reading it needs no copy and no
// synchronisation. Callers read it after a synchronisation (profiler, tuner, ios_run_host, ios_sync)
// or, in ios_run, at the next call (a flag set by any earlier, completed launch is reported then).
void check_err(DeviceState& d) {
  if (!d.err) return;
  volatile int* f = d.err;
  if (*f) {
    *f = 0;
    IOS_FAIL(IOS_ERR_KERNEL, "in-kernel dependency wait timed out (a stage's CTAs were not co-resident, or a "
                             "producer never signalled); outputs of that run are invalid");
  }
}

void sync_and_check(Graph& g, cudaStream_t st) {
  if (!g.dev || !g.dev->ready) return;
  IOS_CHECK_CUDA(cudaStreamSynchronize(st));
  IOS_CHECK_CUDA(cudaStreamSynchronize(g.dev->stream));
  check_err(*g.dev);
}

namespace {
// A stream-captured CUDA graph (owned; destroyed with the object).
struct GraphExec {
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  GraphExec() = default;
  GraphExec(const GraphExec&) = delete;
  GraphExec(GraphExec&& o) noexcept : graph(o.graph), exec(o.exec) { o.graph = nullptr; o.exec = nullptr; }
  ~GraphExec() {
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
  }
};
template <class F>
GraphExec capture(DeviceState& d, F&& body) {
  GraphExec g;
  IOS_CHECK_CUDA(cudaStreamBeginCapture(d.stream, cudaStreamCaptureModeThreadLocal));
  try {
    body();
  } catch (...) {
    cudaGraph_t junk = nullptr;
    cudaStreamEndCapture(d.stream, &junk);
    if (junk) cudaGraphDestroy(junk);
    throw;
  }
  IOS_CHECK_CUDA(cudaStreamEndCapture(d.stream, &g.graph));
  IOS_CHECK_CUDA(cudaGraphInstantiate(&g.exec, g.graph, 0));
  return g;
}
}  // namespace

// Stage tuner: every stage of Q is measured under each tiling variant (the profiler protocol of
// ios_stage_latency: warm-up, trials x CUDA-graph reps, median) and keeps the fastest. Stages
// shared by several schedules get one choice. Plans already built with another variant are
// retired (freed with the graph), so schedules captured earlier stay valid.
void tune_schedule(Graph& g, Schedule& q, int trials, int reps) {
  ensure_device(g);
  DeviceState& d = *g.dev;
  for (const Stage& st : q.stages) {
    int bpos = -1;
    const uint64_t mask = g.mask_of(st.ops, &bpos);
    const auto pk = std::make_tuple(bpos, mask, st.strategy);
    if (d.tile_variant.count(pk)) continue;   // tuned for an earlier schedule
    double best = kInf;
    int best_v = 0;
    // variants 0..2 by default; IOS_TUNE_VARIANTS=4 adds the cluster split-K variant (measured: the
    // tuner then picks it for stages it wins in isolation, but the schedule gets slower in context --
    // Inception V3 b=1 0.4915 -> 0.4967-0.5006 ms -- profiles/r2_cluster_split_k.md)
    static const int nv = getenv("IOS_TUNE_VARIANTS") ? std::max(1, std::min(kTileVariants, atoi(getenv("IOS_TUNE_VARIANTS"))))
                                                       : kVariantCluster;
    for (int v = 0; v < nv; ++v) {
      StagePlan* p = nullptr;
      try {
        p = build_plan(g, bpos, mask, st.strategy, v);
      } catch (const Error& e) {
        if (e.code != IOS_ERR_UNSUPPORTED) throw;
        continue;
      }
      double ms = 0.0;
      if (!p->empty) {
        for (int i = 0; i < 3; ++i) launch_plan(p, d.stream);
        GraphExec rep = capture(d, [&] {
          for (int i = 0; i < reps; ++i) launch_plan(p, d.stream);
        });
        std::vector<double> t;
        for (int tr = 0; tr < trials; ++tr) {
          IOS_CHECK_CUDA(cudaEventRecord(d.ev0, d.stream));
          IOS_CHECK_CUDA(cudaGraphLaunch(rep.exec, d.stream));
          IOS_CHECK_CUDA(cudaEventRecord(d.ev1, d.stream));
          IOS_CHECK_CUDA(cudaEventSynchronize(d.ev1));
          float e = 0;
          IOS_CHECK_CUDA(cudaEventElapsedTime(&e, d.ev0, d.ev1));
          t.push_back((double)e / reps);
        }
        check_err(d);
        std::sort(t.begin(), t.end());
        ms = t[t.size() / 2];
      }
      IOS_CHECK_CUDA(cudaStreamSynchronize(d.stream));
      free_plan(d, p);
      if (ms < best) {
        best = ms;
        best_v = v;
      }
    }
    d.tile_variant[pk] = best_v;
    auto it = d.plans.find(pk);
    if (it != d.plans.end()) {   // rebuilt with the chosen variant on next use
      d.retired.push_back(it->second);
      d.plans.erase(it);
      ++d.plan_gen;              // every captured schedule re-captures with the new plan
    }
  }
  destroy_schedule_exec(q);
}

double stage_latency(Graph& g, const std::vector<int>& ops, int strategy, const ios_profile_opts* opts) {
  ensure_device(g);
  DeviceState& d = *g.dev;
  int bpos = -1;
  const uint64_t mask = g.mask_of(ops, &bpos);
  const int warmup = opts && opts->warmup > 0 ? opts->warmup : 10;
  const int trials = opts && opts->trials > 0 ? opts->trials : 5;
  const int reps = opts && opts->reps > 0 ? opts->reps : 20;
  const bool flush = opts && opts->l2_flush;
  // measure with the cached plan if a run already built one, else with a transient plan that is
  // dropped afterwards (the DP measures each distinct stage once; ios_run rebuilds what it needs)
  const auto key = std::make_tuple(g.block_sig(bpos), mask, strategy);
  StagePlan* p;
  bool transient = false;
  auto pit = d.plans.find(std::make_tuple(bpos, mask, strategy));
  try {
    if (pit != d.plans.end()) {
      p = pit->second;
    } else {
      p = build_plan(g, bpos, mask, strategy);
      transient = true;
    }
  } catch (const Error& e) {
    if (e.code != IOS_ERR_UNSUPPORTED) throw;
    g.latency_cache[key] = kInf;   // not executable -> never chosen
    return kInf;
  }
  struct Drop {
    DeviceState& d;
    StagePlan* p;
    bool on;
    ~Drop() {
      if (on) free_plan(d, p);
    }
  } drop{d, p, transient};
  double ms = 0.0;
  if (!p->empty) {
    if (flush && !d.l2buf) d.l2buf = dmalloc(d, (size_t)d.l2bytes);
    for (int i = 0; i < warmup; ++i) launch_plan(p, d.stream);
    // the `reps` back-to-back launches are one CUDA graph, the launch mechanism ios_run uses
    // (the DP must measure stages the way they run)
    GraphExec rep = capture(d, [&] {
      for (int i = 0; i < reps; ++i) launch_plan(p, d.stream);
    });
    std::vector<double> t;
    for (int tr = 0; tr < trials; ++tr) {
      if (flush) IOS_CHECK_CUDA(launch_l2_flush(d.l2buf, d.l2bytes, d.stream));
      IOS_CHECK_CUDA(cudaEventRecord(d.ev0, d.stream));
      IOS_CHECK_CUDA(cudaGraphLaunch(rep.exec, d.stream));
      IOS_CHECK_CUDA(cudaEventRecord(d.ev1, d.stream));
      IOS_CHECK_CUDA(cudaEventSynchronize(d.ev1));
      float e = 0;
      IOS_CHECK_CUDA(cudaEventElapsedTime(&e, d.ev0, d.ev1));
      t.push_back((double)e / reps);
    }
    check_err(d);
    std::sort(t.begin(), t.end());
    ms = t[t.size() / 2];
  }
  g.latency_cache[key] = ms;
  return ms;
}

// Search-time profiling (Z15, batched): per batch of up to 48 transient plans, one warm-up launch
// each, then `trials` rounds of `reps` back-to-back launches per plan between CUDA events, a
// single host sync per batch; median over rounds of the per-launch mean.
void measure_stages(Graph& g, int bpos, const std::vector<std::pair<uint64_t, int>>& stages) {
  if (stages.empty()) return;
  ensure_device(g);
  DeviceState& d = *g.dev;
  // 3 trials x 10 back-to-back launches per stage: with 3 x 3 the DP's choices between schedules
  // whose totals differed by ~1 % were decided by event-timer noise (SqueezeNet r1: DP 165 us vs
  // greedy 160 us when re-measured with the full protocol). Blocks with more than 5000 candidate
  // stages (NASNet cells, RandWire stages) keep 3 launches, bounding the search time; the measured
  // refinement (ios_schedule_refine) re-checks the result in context. IOS_SEARCH_REPS overrides.
  static const int env_reps = getenv("IOS_SEARCH_REPS") ? std::max(1, atoi(getenv("IOS_SEARCH_REPS"))) : 0;
  const int kReps = env_reps ? env_reps : (stages.size() > 5000 ? 3 : 10);
  constexpr int kBatch = 48, kTrials = 3;
  const uint64_t sig = g.block_sig(bpos);
  std::vector<cudaEvent_t> ev;
  auto event = [&](size_t i) {
    while (ev.size() <= i) {
      cudaEvent_t e;
      IOS_CHECK_CUDA(cudaEventCreate(&e));
      ev.push_back(e);
    }
    return ev[i];
  };
  struct Guard {
    std::vector<cudaEvent_t>& ev;
    ~Guard() {
      for (auto e : ev) cudaEventDestroy(e);
    }
  } guard{ev};
  for (size_t b0 = 0; b0 < stages.size(); b0 += kBatch) {
    const size_t b1 = std::min(stages.size(), b0 + kBatch);
    std::vector<StagePlan*> plans(b1 - b0, nullptr);
    struct Drop {
      DeviceState& d;
      std::vector<StagePlan*>& ps;
      ~Drop() {
        for (auto* p : ps) free_plan(d, p);
      }
    } drop{d, plans};
    for (size_t i = b0; i < b1; ++i) {
      const auto& [mask, t] = stages[i];
      try {
        plans[i - b0] = build_plan(g, bpos, mask, t);
      } catch (const Error& e) {
        if (e.code != IOS_ERR_UNSUPPORTED) throw;
        g.latency_cache[std::make_tuple(sig, mask, t)] = kInf;
      }
    }
    for (size_t i = 0; i < 2 * kTrials * kBatch; ++i) event(i);
    // warm-up + all trials of the batch as ONE CUDA graph (event-record nodes around each plan's
    // launches): stages are timed under the launch mechanism ios_run uses
    GraphExec batch = capture(d, [&] {
      for (auto* p : plans)
        if (p) launch_plan(p, d.stream);   // warm-up
      for (int tr = 0; tr < kTrials; ++tr)
        for (size_t i = 0; i < plans.size(); ++i) {
          if (!plans[i] || plans[i]->empty) continue;
          // External: a captured record becomes a real event-record node (not a capture join)
          IOS_CHECK_CUDA(cudaEventRecordWithFlags(ev[2 * (tr * kBatch + i)], d.stream, cudaEventRecordExternal));
          for (int r = 0; r < kReps; ++r) launch_plan(plans[i], d.stream);
          IOS_CHECK_CUDA(cudaEventRecordWithFlags(ev[2 * (tr * kBatch + i) + 1], d.stream, cudaEventRecordExternal));
        }
    });
    IOS_CHECK_CUDA(cudaGraphLaunch(batch.exec, d.stream));
    IOS_CHECK_CUDA(cudaStreamSynchronize(d.stream));
    check_err(d);
    for (size_t i = 0; i < plans.size(); ++i) {
      if (!plans[i]) continue;
      const auto& [mask, t] = stages[b0 + i];
      double ms = 0.0;
      if (!plans[i]->empty) {
        std::vector<double> v;
        for (int tr = 0; tr < kTrials; ++tr) {
          float e = 0;
          IOS_CHECK_CUDA(cudaEventElapsedTime(&e, ev[2 * (tr * kBatch + i)], ev[2 * (tr * kBatch + i) + 1]));
          v.push_back((double)e / kReps);
        }
        std::sort(v.begin(), v.end());
        ms = v[v.size() / 2];
      }
      g.latency_cache[std::make_tuple(sig, mask, t)] = ms;
    }
  }
}

int stage_trace(Graph& g, const std::vector<int>& ops, int strategy, uint64_t* out, int cap) {
  ensure_device(g);
  DeviceState& d = *g.dev;
  int bpos = -1;
  const uint64_t mask = g.mask_of(ops, &bpos);
  StagePlan* p = get_plan(g, bpos, mask, strategy);
  if (p->empty) return 0;
  launch_plan(p, d.stream);                        // warm
  const size_t n = (size_t)p->grid * 16;
  uint64_t* buf = static_cast<uint64_t*>(dmalloc(d, n * sizeof(uint64_t)));
  StageDesc sd = p->sd;
  sd.trace = (uint64_t)buf;
  // the traced (F_TRACE) instantiation runs once untimed first: its code is then in the SMs'
  // instruction caches like the production kernel's is in back-to-back runs (IOS_TRACE_COLD=1 skips)
  static const bool cold = getenv("IOS_TRACE_COLD") && atoi(getenv("IOS_TRACE_COLD")) != 0;
  if (!cold) IOS_CHECK_CUDA(launch_stage(sd, p->dtype, p->grid, d.stream));
  IOS_CHECK_CUDA(launch_stage(sd, p->dtype, p->grid, d.stream));
  IOS_CHECK_CUDA(cudaStreamSynchronize(d.stream));
  std::vector<uint64_t> h(n);
  IOS_CHECK_CUDA(cudaMemcpy(h.data(), buf, n * sizeof(uint64_t), cudaMemcpyDeviceToHost));
  for (size_t i = 0; i < n && i < (size_t)cap; ++i) out[i] = h[i];
  return p->grid;
}

void run_schedule(Graph& g, Schedule& q, const void* d_in, void* d_out, cudaStream_t st) {
  ensure_device(g);
  DeviceState& d = *g.dev;
  check_err(d);   // a dependency-wait timeout in an earlier (completed) run
  if (!q.exec || q.exec_in != d_in || q.exec_out != d_out || q.exec_gen != d.plan_gen) {
    destroy_schedule_exec(q);
    std::vector<StagePlan*> plans;
    for (const Stage& s : q.stages) {
      int bpos = -1;
      const uint64_t mask = g.mask_of(s.ops, &bpos);
      plans.push_back(get_plan(g, bpos, mask, s.strategy));
    }
    // plans are built on the library's stream (pool allocations, descriptor / weight / tensor-map
    // uploads, counter memsets): they must be complete before the caller's stream runs them
    IOS_CHECK_CUDA(cudaStreamSynchronize(d.stream));
    const Op& in = g.ops[0];
    const Op& last = g.ops.back();
    IOS_CHECK_CUDA(cudaStreamBeginCapture(d.stream, cudaStreamCaptureModeThreadLocal));
    int launches = 0;
    cudaError_t e = launch_nchw_to_nhwc(static_cast<const float*>(d_in), d.od[0].out, g.dtype(), in.N, in.C, d.stream);
    ++launches;
    if (e == cudaSuccess && d.unfold) {
      e = launch_nchw_unfold(static_cast<const float*>(d_in), d.unfold_view, g.dtype(), in.N, in.C, in.W, d.unfold_kw,
                             d.unfold_sw, d.unfold_pw, d.stream);
      ++launches;
    }
    for (StagePlan* p : plans) {
      if (e != cudaSuccess) break;
      if (p->empty) continue;
      e = launch_stage(p->sd, p->dtype, p->grid, d.stream);
      ++launches;
    }
    if (e == cudaSuccess) {
      e = launch_nhwc_to_nchw(d.od[last.id].out, g.dtype(), static_cast<float*>(d_out), last.N, last.C, d.stream);
      ++launches;
    }
    cudaGraph_t graph = nullptr;
    cudaError_t e2 = cudaStreamEndCapture(d.stream, &graph);
    if (e != cudaSuccess) {
      if (graph) cudaGraphDestroy(graph);
      IOS_CHECK_CUDA(e);
    }
    IOS_CHECK_CUDA(e2);
    q.graph = graph;
    IOS_CHECK_CUDA(cudaGraphInstantiate(&q.exec, graph, 0));
    q.exec_in = d_in;
    q.exec_out = d_out;
    q.exec_gen = d.plan_gen;
    q.n_launches = launches;
  }
  IOS_CHECK_CUDA(cudaGraphLaunch(q.exec, st));
}

// In-run stage timeline (A7 "in context"): Q exactly as ios_run executes it (one CUDA graph, PDL
// between stage launches), except that every stage launch records the earliest start (after its
// PDL wait) and the latest exit of its CTAs on %globaltimer. A stage's *attributable* time is its
// end minus the previous stage's end (stage 0: minus its own start), so the attributable times sum
// to the whole schedule's span and overlap through PDL is charged to the stage that hides it.
// `reps` runs, each optionally after an L2 flush (the bench's protocol); per stage the mean over
// reps of (start, end) relative to stage 0's start, and of the attributable time, in us.
void run_timeline(Graph& g, Schedule& q, const void* d_in, void* d_out, int reps, bool flush,
                  std::vector<double>& out) {
  ensure_device(g);
  DeviceState& d = *g.dev;
  check_err(d);
  const int n = (int)q.stages.size();
  std::vector<StagePlan*> plans;
  for (const Stage& s : q.stages) {
    int bpos = -1;
    const uint64_t mask = g.mask_of(s.ops, &bpos);
    plans.push_back(get_plan(g, bpos, mask, s.strategy));
  }
  std::vector<void*> tmp;
  struct Free {
    DeviceState& d;
    std::vector<void*>& v;
    ~Free() {
      cudaStreamSynchronize(d.stream);
      for (void* p : v) cudaFreeAsync(p, d.stream);
    }
  } fr{d, tmp};
  uint64_t* stamps = static_cast<uint64_t*>(dmalloc(d, (size_t)n * 2 * sizeof(uint64_t), &tmp));
  if (flush && !d.l2buf) d.l2buf = dmalloc(d, (size_t)d.l2bytes);
  IOS_CHECK_CUDA(cudaStreamSynchronize(d.stream));
  GraphExec ex = capture(d, [&] {
    // starts = UINT64_MAX (atomicMin), ends = 0 (atomicMax): even slots 0xFF.., odd slots 0
    for (int i = 0; i < n; ++i) {
      IOS_CHECK_CUDA(cudaMemsetAsync(stamps + 2 * i, 0xFF, sizeof(uint64_t), d.stream));
      IOS_CHECK_CUDA(cudaMemsetAsync(stamps + 2 * i + 1, 0, sizeof(uint64_t), d.stream));
    }
    const Op& in = g.ops[0];
    IOS_CHECK_CUDA(launch_nchw_to_nhwc(static_cast<const float*>(d_in), d.od[0].out, g.dtype(), in.N, in.C, d.stream));
    if (d.unfold)
      IOS_CHECK_CUDA(launch_nchw_unfold(static_cast<const float*>(d_in), d.unfold_view, g.dtype(), in.N, in.C, in.W,
                                        d.unfold_kw, d.unfold_sw, d.unfold_pw, d.stream));
    for (int i = 0; i < n; ++i) {
      if (plans[i]->empty) continue;
      StageDesc sd = plans[i]->sd;
      sd.stamp = (uint64_t)(stamps + 2 * i);
      IOS_CHECK_CUDA(launch_stage(sd, plans[i]->dtype, plans[i]->grid, d.stream));
    }
    const Op& last = g.ops.back();
    IOS_CHECK_CUDA(launch_nhwc_to_nchw(d.od[last.id].out, g.dtype(), static_cast<float*>(d_out), last.N, last.C, d.stream));
  });
  out.assign((size_t)n * 3, 0.0);
  std::vector<uint64_t> h((size_t)n * 2);
  for (int r = 0; r < reps; ++r) {
    if (flush) IOS_CHECK_CUDA(launch_l2_flush(d.l2buf, d.l2bytes, d.stream));
    IOS_CHECK_CUDA(cudaGraphLaunch(ex.exec, d.stream));
    IOS_CHECK_CUDA(cudaStreamSynchronize(d.stream));
    check_err(d);
    IOS_CHECK_CUDA(cudaMemcpy(h.data(), stamps, h.size() * sizeof(uint64_t), cudaMemcpyDeviceToHost));
    uint64_t t0 = 0;
    for (int i = 0; i < n && !t0; ++i)
      if (!plans[i]->empty) t0 = h[2 * i];
    double prev_end = 0.0;
    for (int i = 0; i < n; ++i) {
      double st = prev_end, en = prev_end;
      if (!plans[i]->empty) {
        st = (double)(int64_t)(h[2 * i] - t0) * 1e-3;
        en = (double)(int64_t)(h[2 * i + 1] - t0) * 1e-3;
      }
      out[3 * i] += st / reps;
      out[3 * i + 1] += en / reps;
      out[3 * i + 2] += (en - prev_end) / reps;
      prev_end = en;
    }
  }
}

// Tuned tiling variants (ios_schedule_tune's choices) as text, one "block_pos mask strategy variant"
// per line, so a profiler run (tools/ncu_run.py) replays exactly the plans the bench timed.
void save_tile_variants(Graph& g, const std::string& path) {
  ensure_device(g);
  std::ofstream f(path);
  if (!f) IOS_FAIL(IOS_ERR_INVALID_ARG, "cannot write " + path);
  f << "ios-tile-variants v1 ops=" << g.ops.size() << " batch=" << g.batch << " math=" << (int)g.math << "\n";
  for (auto& [k, v] : g.dev->tile_variant)
    f << std::get<0>(k) << " " << std::get<1>(k) << " " << std::get<2>(k) << " " << v << "\n";
}

void load_tile_variants(Graph& g, const std::string& path) {
  ensure_device(g);
  DeviceState& d = *g.dev;
  std::ifstream f(path);
  if (!f) IOS_FAIL(IOS_ERR_INVALID_ARG, "cannot read " + path);
  std::string head;
  std::getline(f, head);
  std::ostringstream want;
  want << "ios-tile-variants v1 ops=" << g.ops.size() << " batch=" << g.batch << " math=" << (int)g.math;
  if (head != want.str()) IOS_FAIL(IOS_ERR_INVALID_ARG, "tile variants belong to another graph");
  long long bp, t, v;
  unsigned long long m;
  while (f >> bp >> m >> t >> v) {
    if (bp < 0 || bp >= (long long)g.blocks.size() || v < 0 || v >= kTileVariants)
      IOS_FAIL(IOS_ERR_INVALID_ARG, "malformed tile variant entry");
    const auto key = std::make_tuple((int)bp, (uint64_t)m, (int)t);
    d.tile_variant[key] = (int)v;
    auto it = d.plans.find(key);
    if (it != d.plans.end()) {
      d.retired.push_back(it->second);
      d.plans.erase(it);
      ++d.plan_gen;
    }
  }
  if (!f.eof()) IOS_FAIL(IOS_ERR_INVALID_ARG, "malformed tile variant file");
}

int schedule_launches(Graph& g, Schedule& q) {
  ensure_device(g);
  int n = 2 + (g.dev->unfold ? 1 : 0);
  for (const Stage& s : q.stages) {
    int bpos = -1;
    const uint64_t mask = g.mask_of(s.ops, &bpos);
    if (!get_plan(g, bpos, mask, s.strategy)->empty) ++n;
  }
  return n;
}

void op_output(Graph& g, int op, void* d_out, cudaStream_t st) {
  ensure_device(g);
  const Op& o = g.ops[op];
  IOS_CHECK_CUDA(launch_nhwc_to_nchw(g.dev->od[op].out, g.dtype(), static_cast<float*>(d_out), o.N, o.C, st));
}

void destroy_schedule_exec(Schedule& q) {
  if (q.exec) cudaGraphExecDestroy(q.exec);
  if (q.graph) cudaGraphDestroy(q.graph);
  q.exec = nullptr;
  q.graph = nullptr;
}

void destroy_device(Graph& g) {
  if (!g.dev) return;
  DeviceState& d = *g.dev;
  if (d.ready) cudaDeviceSynchronize();   // callers' streams may still run this graph's stages
  for (auto& [k, p] : d.plans) free_plan(d, p);
  for (StagePlan* p : d.retired) free_plan(d, p);
  if (d.stream) cudaStreamSynchronize(d.stream);
  for (void* p : d.allocs) cudaFree(p);
  if (d.err) cudaFreeHost(d.err);
  if (d.ev0) cudaEventDestroy(d.ev0);
  if (d.ev1) cudaEventDestroy(d.ev1);
  if (d.stream) cudaStreamDestroy(d.stream);
  delete g.dev;
  g.dev = nullptr;
}

}  // namespace ios
