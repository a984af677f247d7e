// Persistent grouped stage kernel for sm_100a.
//
// ONE launch runs every member op of a stage: all groups of a concurrent stage, or the
// single merged convolution of a merge stage. The stage is a list of "problems"
// (GEMM-shaped convs and memory-bound SIMT ops) whose tiles are laid out so every dependency
// points backwards; CTA c takes tiles c, c + grid, ... (static round robin). Intra-group
// sequencing is a wait on per-problem completion counters; because every CTA is resident
// and walks its tiles in increasing order, the lowest unfinished tile can always progress.
//
// Warp roles (one CTA per SM, 288 threads):
//   warps 0-3  producers: implicit-im2col gather of A (cp.async 16 B pieces, zero fill for padding
//              and ragged M/K) + the weight chunk B via one cp.async.bulk (TMA engine)
//   warp  8    tcgen05.mma issuer (kind::tf32 or kind::f16/bf16), fp32 accumulators in TMEM,
//              double-buffered (2 x 256 columns)
//   warps 4-7  epilogue: tcgen05.ld -> bias -> ReLU -> store into each branch's channel slice
//              (concat addressing: the split of a merged conv and the concat are free);
//              deterministic split-K fix-up by the last-arriving tile; SIMT tiles (pool, add,
//              concat copy, depthwise) run here too.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <cstdio>

#include "stage_desc.h"

namespace ios {

// ------------------------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t a, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(a),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t a) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint32_t a, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t mbar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(mbar)
      : "memory");
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void named_bar(int id, int n) {
  __syncwarp();   // bar.sync is .aligned: reconverge lanes that diverged (e.g. one lane spun on a counter)
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// UMMA shared-memory matrix descriptor, K-major, SWIZZLE_NONE: core matrices of 8 rows x 16 B;
// LBO = byte distance between K-adjacent core matrices, SBO = between 8-row groups (sm_100 version 1).
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}
// Instruction descriptor: D f32, A/B = tf32 (2) or bf16 (1), K-major both, N >> 3, M >> 4.
__device__ __forceinline__ uint32_t umma_idesc(int bf16, int n) {
  const uint32_t f = bf16 ? 1u : 2u;
  return (1u << 4) | (f << 7) | (f << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(kBM >> 4) << 24);
}
template <int DT>
__device__ __forceinline__ void umma(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  if constexpr (DT == ET_BF16)
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
  else
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .b32 r;\n\t.reg .pred p;\n\telect.sync r|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(pred));
  return pred != 0;
}
__device__ __forceinline__ void umma_commit(uint32_t mbar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(mbar) : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  __syncwarp();   // tcgen05.ld is .sync.aligned
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr)
      : "memory");
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ float tf32_round(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// ------------------------------------------------------------------------------- element access
// 16-byte vectors: 4 fp32 or 8 bf16 channels. All views have 16 B-aligned pixels/channel offsets.
struct Vec8 {
  float v[8];
};

__device__ __forceinline__ void load_vec(const View& vw, int dtype, int64_t pix, int c, float* out, int nv) {
  // nv = elements per 16 B (4 fp32 / 8 bf16); cache-global loads (other CTAs wrote these in this launch)
  if (dtype == ET_F32) {
    const float4* p = reinterpret_cast<const float4*>(reinterpret_cast<const float*>(vw.ptr) + pix * vw.cstride + vw.coff + c);
    float4 a = __ldcg(p);
    out[0] = a.x; out[1] = a.y; out[2] = a.z; out[3] = a.w;
  } else {
    const uint4* p = reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(vw.ptr) + pix * vw.cstride + vw.coff + c);
    uint4 a = __ldcg(p);
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&a);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float2 f = __bfloat1622float2(h[i]);
      out[2 * i] = f.x;
      out[2 * i + 1] = f.y;
    }
  }
}

__device__ __forceinline__ void store_vec(const View& vw, int dtype, int64_t pix, int c, const float* in) {
  if (dtype == ET_F32) {
    float4 a = make_float4(tf32_round(in[0]), tf32_round(in[1]), tf32_round(in[2]), tf32_round(in[3]));
    *reinterpret_cast<float4*>(reinterpret_cast<float*>(vw.ptr) + pix * vw.cstride + vw.coff + c) = a;
  } else {
    uint4 a;
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&a);
#pragma unroll
    for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(in[2 * i], in[2 * i + 1]);
    *reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(vw.ptr) + pix * vw.cstride + vw.coff + c) = a;
  }
}

__device__ __forceinline__ float load_elem(const View& vw, int dtype, int64_t pix, int c) {
  if (dtype == ET_F32) return __ldcg(reinterpret_cast<const float*>(vw.ptr) + pix * vw.cstride + vw.coff + c);
  const unsigned short* p = reinterpret_cast<const unsigned short*>(vw.ptr) + pix * vw.cstride + vw.coff + c;
  unsigned short u = __ldcg(p);
  return __uint_as_float(((uint32_t)u) << 16);
}
__device__ __forceinline__ void store_elem(const View& vw, int dtype, int64_t pix, int c, float x) {
  if (dtype == ET_F32)
    reinterpret_cast<float*>(vw.ptr)[pix * vw.cstride + vw.coff + c] = tf32_round(x);
  else
    reinterpret_cast<__nv_bfloat16*>(vw.ptr)[pix * vw.cstride + vw.coff + c] = __float2bfloat16_rn(x);
}

// ------------------------------------------------------------------------------ dependency waits
__device__ __forceinline__ void wait_deps(const Problem& P, int* counters, int* err) {
  for (int d = 0; d < P.n_deps; ++d) {
    const int* c = counters + P.dep_idx[d];
    const int target = P.dep_target[d];
    long long t0 = clock64();
    while (ld_acquire(c) < target) {
      __nanosleep(64);
      if (clock64() - t0 > (long long)8000000000LL) {   // ~4 s: deadlock guard -> IOS_ERR_KERNEL
        atomicExch(err, 1);
        break;
      }
    }
  }
}

// -------------------------------------------------------------------------------- SIMT tile body
// Runs on the 128 epilogue threads. Items are output pixels x 16 B channel vectors.
__device__ void simt_tile(const Problem& P, const View* views, int tile, int tid) {
  const int dtype = P.dtype;
  const int nv = dtype == ET_F32 ? 4 : 8;
  const View& out = P.out;
  const int nvec = out.C / nv;
  const int item0 = tile * P.items_per_tile;
  const int item1 = min(item0 + P.items_per_tile, P.n_items);
  if (P.kind == PK_GAVGPOOL) {
    // items = (image, channel vector); reduce over H*W
    const View& in = views[P.in_begin];
    const int hw = in.H * in.W;
    const float inv = 1.0f / (float)hw;
    for (int idx = item0 + tid; idx < item1; idx += 128) {
      const int n = idx / nvec, v = idx % nvec;
      float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      for (int p = 0; p < hw; ++p) {
        float x[8];
        load_vec(in, dtype, (int64_t)n * hw + p, v * nv, x, nv);
#pragma unroll
        for (int e = 0; e < 8; ++e)
          if (e < nv) acc[e] += (P.flags & 2) ? fmaxf(x[e], 0.f) : x[e];
      }
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[e] *= inv;
      store_vec(out, dtype, n, v * nv, acc);
    }
    return;
  }
  const int total = (item1 - item0) * nvec;
  const int HoWo = P.Ho * P.Wo;
  for (int idx = tid; idx < total; idx += 128) {
    const int pix = item0 + idx / nvec;       // output pixel (n, oh, ow)
    const int c = (idx % nvec) * nv;
    const int n = pix / HoWo;
    const int rem = pix - n * HoWo;
    const int oh = rem / P.Wo, ow = rem - (rem / P.Wo) * P.Wo;
    float acc[8];
    switch (P.kind) {
      case PK_ADD: {
        const float* aw = reinterpret_cast<const float*>(P.add_w);
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[e] = 0.f;
        for (int i = 0; i < P.n_in; ++i) {
          float x[8];
          load_vec(views[P.in_begin + i], dtype, pix, c, x, nv);
          const float w = aw ? aw[i] : 1.0f;
#pragma unroll
          for (int e = 0; e < 8; ++e) acc[e] = fmaf(w, x[e], acc[e]);
        }
        break;
      }
      case PK_MAXPOOL:
      case PK_AVGPOOL: {
        const View& in = views[P.in_begin];
        const bool is_max = P.kind == PK_MAXPOOL;
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[e] = is_max ? -INFINITY : 0.f;
        const int hs = oh * P.sh - P.ph, ws = ow * P.sw - P.pw;
        for (int i = 0; i < P.kh; ++i) {
          const int ih = hs + i;
          if (ih < 0 || ih >= in.H) continue;
          for (int j = 0; j < P.kw; ++j) {
            const int iw = ws + j;
            if (iw < 0 || iw >= in.W) continue;
            float x[8];
            load_vec(in, dtype, ((int64_t)n * in.H + ih) * in.W + iw, c, x, nv);
#pragma unroll
            for (int e = 0; e < 8; ++e) acc[e] = is_max ? fmaxf(acc[e], x[e]) : acc[e] + x[e];
          }
        }
        if (!is_max) {
          // divisor: window clipped to the padded input (include pad) or to the input (exclude pad)
          const int he = min(hs + P.kh, in.H + P.ph), we = min(ws + P.kw, in.W + P.pw);
          int div;
          if (P.flags & 8) div = (he - hs) * (we - ws);
          else div = (min(he, in.H) - max(hs, 0)) * (min(we, in.W) - max(ws, 0));
          const float inv = 1.0f / (float)div;
#pragma unroll
          for (int e = 0; e < 8; ++e) acc[e] *= inv;
        }
        break;
      }
      case PK_DWCONV: {
        // ReLU(sum_i w_i x_i) -> depthwise k x k; weights fp32 [C][kh*kw]
        const float* wd = reinterpret_cast<const float*>(P.wts);
        const float* aw = reinterpret_cast<const float*>(P.add_w);
        const View& in0 = views[P.in_begin];
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[e] = 0.f;
        const int hs = oh * P.sh - P.ph, ws = ow * P.sw - P.pw;
        const int kk = P.kh * P.kw;
        for (int i = 0; i < P.kh; ++i) {
          const int ih = hs + i;
          if (ih < 0 || ih >= in0.H) continue;
          for (int j = 0; j < P.kw; ++j) {
            const int iw = ws + j;
            if (iw < 0 || iw >= in0.W) continue;
            const int64_t ipix = ((int64_t)n * in0.H + ih) * in0.W + iw;
            float a[8] = {0, 0, 0, 0, 0, 0, 0, 0};
            for (int s = 0; s < P.n_in; ++s) {
              float x[8];
              load_vec(views[P.in_begin + s], dtype, ipix, c, x, nv);
              const float w = aw ? aw[s] : 1.0f;
#pragma unroll
              for (int e = 0; e < 8; ++e) a[e] = fmaf(w, x[e], a[e]);
            }
            const int tap = i * P.kw + j;
#pragma unroll
            for (int e = 0; e < 8; ++e)
              if (e < nv) acc[e] = fmaf(wd[(c + e) * kk + tap], fmaxf(a[e], 0.f), acc[e]);
          }
        }
        break;
      }
      case PK_COPY:
      default: {
        // concat gather (element-wise: inputs may have channel counts that are not vector multiples)
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          acc[e] = 0.f;
          if (e >= nv) continue;
          int ch = c + e, off = 0;
          for (int i = 0; i < P.n_in; ++i) {
            const View& vi = views[P.in_begin + i];
            const int ci = vi.Cl;
            if (ch < off + ci) {
              acc[e] = load_elem(vi, dtype, pix, ch - off);
              break;
            }
            off += ci;
          }
        }
        break;
      }
    }
    store_vec(out, dtype, pix, c, acc);
  }
}


// --------------------------------------------------------------------------------- the kernel
struct Ring {          // smem ring iterator (slot, phase)
  int slot = 0;
  uint32_t phase = 0;
  __device__ __forceinline__ void next() {
    if (++slot == kStages) {
      slot = 0;
      phase ^= 1u;
    }
  }
};

__device__ __forceinline__ int find_problem(const int* sm_tile_begin, int n_problems, int tile, int hint) {
  int p = hint;
  while (p + 1 < n_problems && sm_tile_begin[p + 1] <= tile) ++p;
  return p;
}

template <int DT>
__global__ void __launch_bounds__(kThreads, 1) ios_stage_kernel(const StageDesc sd) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;                                       // kStages x 16 KB
  uint8_t* sB = smem + kStages * kAStageBytes;              // kStages x 32 KB
  uint64_t* bars = reinterpret_cast<uint64_t*>(sB + kStages * kBStageBytes);
  uint64_t* full = bars;                                    // [kStages]
  uint64_t* empty = bars + kStages;                         // [kStages]
  uint64_t* tfull = bars + 2 * kStages;                     // [2]
  uint64_t* tempty = bars + 2 * kStages + 2;                // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kStages + 4);
  int* flag = reinterpret_cast<int*>(tmem_slot + 1);
  __shared__ int sm_tile_begin[kMaxProblems];

  const Problem* probs = reinterpret_cast<const Problem*>(sd.problems);
  const View* views = reinterpret_cast<const View*>(sd.views);
  const Segment* segs = reinterpret_cast<const Segment*>(sd.segs);
  int* counters = reinterpret_cast<int*>(sd.counters);
  int* err = reinterpret_cast<int*>(sd.err);
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;

  for (int i = tid; i < sd.n_problems; i += kThreads) sm_tile_begin[i] = probs[i].tile_begin;
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(smem_u32(&full[s]), kProducerWarps * 32 + 1);
      mbar_init(smem_u32(&empty[s]), 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(smem_u32(&tfull[s]), 1);
      mbar_init(smem_u32(&tempty[s]), 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kMmaWarp && sd.has_gemm) {
    __syncwarp();
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp < kProducerWarps) {
    // ============================================================== PRODUCER (A gather + B bulk)
    const int ptid = tid;                       // 0..127
    const int rig = lane & 7;                   // row inside an 8-row core-matrix group
    const int pc0 = lane >> 3;                  // pieces pc0 and pc0 + 4 of each 128 B chunk row
    Ring ring;
    int hint = 0;
    for (int t = blockIdx.x; t < sd.n_tiles; t += gridDim.x) {
      hint = find_problem(sm_tile_begin, sd.n_problems, t, hint);
      const Problem& P = probs[hint];
      if (P.kind != PK_GEMM) continue;
      if (ptid == 0) wait_deps(P, counters, err);
      named_bar(1, 128);
      const int local = t - P.tile_begin;
      const int s = local % P.split;
      const int rest = local / P.split;
      const int nt = rest % P.n_tiles_n;
      const int mt = rest / P.n_tiles_n;
      const int c0 = s * P.chunks_per_split;
      const int c1 = min(c0 + P.chunks_per_split, P.k_chunks);
      const View in = views[P.in_begin];
      const int esz = P.dtype == ET_BF16 ? 2 : 4;
      const int vec = 16 / esz;
      const int elems = kChunkBytes / esz;
      const int HoWo = P.Ho * P.Wo;
      const bool relu_pre = (P.flags & 2) != 0;
      // per-row state for the 4 rows this thread gathers
      int ih0[4], iw0[4];
      int64_t rbase[4];
      bool rvalid[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int r = (warp + 4 * j) * 8 + rig;
        const int m = mt * kBM + r;
        rvalid[j] = m < P.M;
        const int mm = rvalid[j] ? m : 0;
        const int n = mm / HoWo;
        const int rem = mm - n * HoWo;
        const int oh = rem / P.Wo, ow = rem - (rem / P.Wo) * P.Wo;
        ih0[j] = oh * P.sh - P.ph;
        iw0[j] = ow * P.sw - P.pw;
        rbase[j] = (int64_t)n * in.H * in.W;
      }
      const uint8_t* wsrc = reinterpret_cast<const uint8_t*>(P.wts);
      // the last n tile may run past the packed rows: copy only those (the rest of the smem tile is
      // stale and only feeds accumulator columns that no output segment covers)
      const uint32_t bbytes = (uint32_t)min(P.BN, P.Npad8 - nt * P.BN) * kChunkBytes;
      int pend[2] = {-1, -1};
      for (int c = c0; c < c1; ++c) {
        mbar_wait(smem_u32(&empty[ring.slot]), ring.phase ^ 1u);
        if (ptid == 0) {
          const uint32_t fb = smem_u32(&full[ring.slot]);
          mbar_arrive_expect_tx(fb, bbytes);
          const uint8_t* src = wsrc + ((int64_t)c * (P.Npad8 >> 3) + (int64_t)nt * (P.BN >> 3)) * 1024;
          bulk_g2s(smem_u32(sB + ring.slot * kBStageBytes), src, bbytes, fb);
        }
        uint8_t* a_st = sA + ring.slot * kAStageBytes;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int pc = pc0 + 4 * h;
          const int k = c * elems + pc * vec;
          const bool kvalid = k < P.K;
          const int tap = k / in.C;
          const int ci = k - tap * in.C;
          const int ki = tap / P.kw, kj = tap - (tap / P.kw) * P.kw;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int r = (warp + 4 * j) * 8 + rig;
            const int ih = ih0[j] + ki, iw = iw0[j] + kj;
            const bool ok = kvalid && rvalid[j] && ih >= 0 && ih < in.H && iw >= 0 && iw < in.W;
            const int64_t eoff = ok ? ((rbase[j] + (int64_t)ih * in.W + iw) * in.cstride + in.coff + ci) : 0;
            const uint8_t* src = reinterpret_cast<const uint8_t*>(in.ptr) + eoff * esz;
            uint8_t* dst = a_st + (r >> 3) * 1024 + pc * 128 + (r & 7) * 16;
            if (!relu_pre) {
              cp_async16(smem_u32(dst), src, ok ? 16u : 0u);
            } else {
              uint4 v = make_uint4(0, 0, 0, 0);
              if (ok) v = __ldcg(reinterpret_cast<const uint4*>(src));
              if (esz == 4) {
                float* f = reinterpret_cast<float*>(&v);
                f[0] = fmaxf(f[0], 0.f); f[1] = fmaxf(f[1], 0.f); f[2] = fmaxf(f[2], 0.f); f[3] = fmaxf(f[3], 0.f);
              } else {
                __nv_bfloat162* hb = reinterpret_cast<__nv_bfloat162*>(&v);
                const __nv_bfloat162 z = __floats2bfloat162_rn(0.f, 0.f);
                hb[0] = __hmax2(hb[0], z); hb[1] = __hmax2(hb[1], z); hb[2] = __hmax2(hb[2], z); hb[3] = __hmax2(hb[3], z);
              }
              *reinterpret_cast<uint4*>(dst) = v;
            }
          }
        }
        cp_async_commit();
        // arrive for the chunk issued two iterations ago (keeps up to 3 chunks of cp.async in flight)
        if (pend[0] >= 0) {
          cp_async_wait<2>();
          fence_proxy_async();
          mbar_arrive(smem_u32(&full[pend[0]]));
        }
        pend[0] = pend[1];
        pend[1] = ring.slot;
        ring.next();
      }
      cp_async_wait<0>();
      fence_proxy_async();
      if (pend[0] >= 0) mbar_arrive(smem_u32(&full[pend[0]]));
      if (pend[1] >= 0) mbar_arrive(smem_u32(&full[pend[1]]));
    }
  } else if (warp == kMmaWarp) {
    // ============================================================== MMA ISSUER
    // The whole warp walks the tiles and waits on the barriers (warp-uniform control flow); one
    // elected lane issues tcgen05.mma / tcgen05.commit.
    if (sd.has_gemm) {
      Ring ring;
      int acc = 0;
      uint32_t acc_phase = 0;
      int hint = 0;
      for (int t = blockIdx.x; t < sd.n_tiles; t += gridDim.x) {
        hint = find_problem(sm_tile_begin, sd.n_problems, t, hint);
        const Problem& P = probs[hint];
        if (P.kind != PK_GEMM) continue;
        const int local = t - P.tile_begin;
        const int s = local % P.split;
        const int c0 = s * P.chunks_per_split;
        const int c1 = min(c0 + P.chunks_per_split, P.k_chunks);
        const uint32_t idesc = umma_idesc(DT == ET_BF16, P.BN);
        mbar_wait(smem_u32(&tempty[acc]), acc_phase ^ 1u);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + (uint32_t)acc * kMaxBN;
        for (int c = c0; c < c1; ++c) {
          mbar_wait(smem_u32(&full[ring.slot]), ring.phase);
          tc_fence_after();
          const uint32_t a0 = smem_u32(sA + ring.slot * kAStageBytes);
          const uint32_t b0 = smem_u32(sB + ring.slot * kBStageBytes);
          __syncwarp();
          if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)   // 4 x 32 B of K per 128 B chunk
              umma<DT>(tmem_d, umma_desc(a0 + kk * 256, 128, 1024), umma_desc(b0 + kk * 256, 128, 1024), idesc,
                       (c > c0 || kk > 0) ? 1u : 0u);
            umma_commit(smem_u32(&empty[ring.slot]));
          }
          __syncwarp();
          ring.next();
        }
        if (elect_one()) umma_commit(smem_u32(&tfull[acc]));
        __syncwarp();
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1u;
      }
    }
  } else {
    // ============================================================== EPILOGUE + SIMT (warps 4-7)
    const int etid = tid - kEpilogueWarp0 * 32;   // 0..127 == TMEM lane == tile row
    const int lane_base = (warp & 3) * 32;        // TMEM lanes this warp may access
    int acc = 0;
    uint32_t acc_phase = 0;
    int hint = 0;
    for (int t = blockIdx.x; t < sd.n_tiles; t += gridDim.x) {
      hint = find_problem(sm_tile_begin, sd.n_problems, t, hint);
      const Problem& P = probs[hint];
      if (P.kind != PK_GEMM) {
        if (etid == 0) wait_deps(P, counters, err);
        named_bar(2, 128);
        simt_tile(P, views, t - P.tile_begin, etid);
        named_bar(2, 128);
        if (etid == 0) {
          __threadfence();
          atomicAdd(counters + P.done_idx, 1);
        }
        continue;
      }
      const int local = t - P.tile_begin;
      const int s = local % P.split;
      const int rest = local / P.split;
      const int nt = rest % P.n_tiles_n;
      const int mt = rest / P.n_tiles_n;
      const int m = mt * kBM + etid;
      const bool valid = m < P.M;
      const int esz_out = P.dtype == ET_BF16 ? 2 : 4;
      const float* bias = reinterpret_cast<const float*>(P.bias);
      mbar_wait(smem_u32(&tfull[acc]), acc_phase);
      tc_fence_after();
      const uint32_t tbase = tmem_base + ((uint32_t)lane_base << 16) + (uint32_t)acc * kMaxBN;
      const int out_tile = mt * P.n_tiles_n + nt;
      if (P.split == 1) {
        for (int c0 = 0; c0 < P.BN; c0 += 16) {
          uint32_t v[16];
          tmem_ld16(tbase + c0, v);
          tmem_ld_wait();
          if (!valid) continue;
#pragma unroll
          for (int g = 0; g < 2; ++g) {
            const int ncol = nt * P.BN + c0 + g * 8;
            for (int q = 0; q < P.n_seg; ++q) {
              const Segment& sg = segs[P.seg_begin + q];
              if (ncol >= sg.n0 && ncol < sg.n1) {
                float o[8];
                const float4 b0 = __ldg(reinterpret_cast<const float4*>(bias + ncol));
                const float4 b1 = __ldg(reinterpret_cast<const float4*>(bias + ncol + 4));
                const float bb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                  o[e] = __uint_as_float(v[g * 8 + e]) + bb[e];
                  if (sg.relu) o[e] = fmaxf(o[e], 0.f);
                }
                store_vec(sg.out, P.dtype, m, ncol - sg.n0, o);
                if (esz_out == 4) store_vec(sg.out, P.dtype, m, ncol - sg.n0 + 4, o + 4);
                break;
              }
            }
          }
        }
        tc_fence_before();
        mbar_arrive(smem_u32(&tempty[acc]));
      } else {
        // split-K: write the fp32 partial, the last arriving split reduces in split order
        float* ws = reinterpret_cast<float*>(P.workspace);
        float* mine = ws + (((int64_t)out_tile * P.split + s) * kBM + etid) * P.BN;
        for (int c0 = 0; c0 < P.BN; c0 += 16) {
          uint32_t v[16];
          tmem_ld16(tbase + c0, v);
          tmem_ld_wait();
#pragma unroll
          for (int q = 0; q < 16; q += 4)
            __stcg(reinterpret_cast<float4*>(mine + c0 + q),
                   make_float4(__uint_as_float(v[q]), __uint_as_float(v[q + 1]), __uint_as_float(v[q + 2]),
                               __uint_as_float(v[q + 3])));
        }
        tc_fence_before();
        mbar_arrive(smem_u32(&tempty[acc]));
        __threadfence();
        named_bar(2, 128);
        if (etid == 0) {
          const int old = atomicAdd(counters + P.tilectr_idx + out_tile, 1);
          *flag = (old == P.split - 1);
        }
        named_bar(2, 128);
        const bool last = *flag != 0;
        if (last) {
          __threadfence();
          if (valid) {
            for (int c0 = 0; c0 < P.BN; c0 += 8) {
              const int ncol = nt * P.BN + c0;
              const Segment* sgp = nullptr;
              for (int q = 0; q < P.n_seg; ++q) {
                const Segment& sg = segs[P.seg_begin + q];
                if (ncol >= sg.n0 && ncol < sg.n1) {
                  sgp = &sg;
                  break;
                }
              }
              if (!sgp) continue;
              float o[8] = {0, 0, 0, 0, 0, 0, 0, 0};
              for (int ss = 0; ss < P.split; ++ss) {
                const float* src = ws + (((int64_t)out_tile * P.split + ss) * kBM + etid) * P.BN + c0;
                const float4 x0 = __ldcg(reinterpret_cast<const float4*>(src));
                const float4 x1 = __ldcg(reinterpret_cast<const float4*>(src + 4));
                o[0] += x0.x; o[1] += x0.y; o[2] += x0.z; o[3] += x0.w;
                o[4] += x1.x; o[5] += x1.y; o[6] += x1.z; o[7] += x1.w;
              }
              const float4 b0 = __ldg(reinterpret_cast<const float4*>(bias + ncol));
              const float4 b1 = __ldg(reinterpret_cast<const float4*>(bias + ncol + 4));
              const float bb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
              for (int e = 0; e < 8; ++e) {
                o[e] += bb[e];
                if (sgp->relu) o[e] = fmaxf(o[e], 0.f);
              }
              store_vec(sgp->out, P.dtype, m, ncol - sgp->n0, o);
              if (esz_out == 4) store_vec(sgp->out, P.dtype, m, ncol - sgp->n0 + 4, o + 4);
            }
          }
        }
        if (!last) {
          acc ^= 1;
          if (acc == 0) acc_phase ^= 1u;
          continue;
        }
      }
      named_bar(2, 128);
      if (etid == 0) {
        __threadfence();
        atomicAdd(counters + P.done_idx, 1);
      }
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1u;
    }
  }

  // ---------------------------------------------------------------------------- teardown
  __syncwarp();   // the MMA warp ran its loop on lane 0 only
  tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp && sd.has_gemm) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(kTmemCols) : "memory");
  }
  if (tid == 0) {
    // the last CTA out resets the stage's counters for the next launch (graph-replay safe)
    __threadfence();
    const int old = atomicAdd(counters, 1);
    if (old == (int)gridDim.x - 1) {
      __threadfence();
      for (int i = 1; i < sd.n_counters; ++i) counters[i] = 0;
      __threadfence();
      counters[0] = 0;
    }
  }
}

// ------------------------------------------------------------------------ boundary layout kernels
// NCHW fp32 (caller) -> NHWC padded (internal); rounds to the storage precision (Z14).
__global__ void nchw_to_nhwc_kernel(const float* __restrict__ in, View out, int dtype, int N, int C) {
  const int64_t total = (int64_t)N * out.H * out.W * out.C;
  const int64_t hw = (int64_t)out.H * out.W;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i % out.C);
    const int64_t pix = i / out.C;
    const int64_t n = pix / hw, p = pix % hw;
    const float x = c < C ? in[(n * C + c) * hw + p] : 0.f;
    store_elem(out, dtype, pix, c, x);
  }
}

__global__ void nhwc_to_nchw_kernel(View in, int dtype, float* __restrict__ out, int N, int C) {
  const int64_t hw = (int64_t)in.H * in.W;
  const int64_t total = (int64_t)N * C * hw;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = i % hw;
    const int64_t nc = i / hw;
    const int c = (int)(nc % C);
    const int64_t n = nc / C;
    out[i] = load_elem(in, dtype, n * hw + p, c);
  }
}

// Writes 2x the L2 size between profiler trials (Z15 l2_flush option).
__global__ void l2_flush_kernel(int4* buf, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    buf[i] = make_int4((int)i, 0, 0, 0);
}

// ------------------------------------------------------------------------------ host launchers
cudaError_t launch_stage(const StageDesc& sd, int dtype, int grid, cudaStream_t st) {
  static bool attr_done = false;
  if (!attr_done) {
    cudaError_t e = cudaFuncSetAttribute(ios_stage_kernel<ET_F32>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes + 1024);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(ios_stage_kernel<ET_BF16>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes + 1024);
    if (e != cudaSuccess) return e;
    attr_done = true;
  }
  if (dtype == ET_BF16)
    ios_stage_kernel<ET_BF16><<<grid, kThreads, kSmemBytes + 1024, st>>>(sd);
  else
    ios_stage_kernel<ET_F32><<<grid, kThreads, kSmemBytes + 1024, st>>>(sd);
  return cudaGetLastError();
}

cudaError_t launch_nchw_to_nhwc(const float* in, const View& out, int dtype, int N, int C, cudaStream_t st) {
  const int64_t total = (int64_t)N * out.H * out.W * out.C;
  int64_t g64 = (total + 255) / 256; int grid = (int)(g64 < 148 * 8 ? g64 : 148 * 8);
  nchw_to_nhwc_kernel<<<grid, 256, 0, st>>>(in, out, dtype, N, C);
  return cudaGetLastError();
}

cudaError_t launch_nhwc_to_nchw(const View& in, int dtype, float* out, int N, int C, cudaStream_t st) {
  const int64_t total = (int64_t)N * C * in.H * in.W;
  int64_t g64 = (total + 255) / 256; int grid = (int)(g64 < 148 * 8 ? g64 : 148 * 8);
  if (grid < 1) grid = 1;
  nhwc_to_nchw_kernel<<<grid, 256, 0, st>>>(in, dtype, out, N, C);
  return cudaGetLastError();
}

cudaError_t launch_l2_flush(void* buf, int64_t bytes, cudaStream_t st) {
  l2_flush_kernel<<<148 * 4, 256, 0, st>>>(reinterpret_cast<int4*>(buf), bytes / 16);
  return cudaGetLastError();
}

}  // namespace ios
