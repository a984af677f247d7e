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
#include <climits>
#include <cstdio>
#include <cstdlib>

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
// ---- cluster split-K (F_CSK): distributed shared memory between the CTAs of a cluster
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t rank) {   // own smem address -> peer's
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// 16 B into a peer CTA's shared memory; the bytes complete_tx on the peer's mbarrier
__device__ __forceinline__ void st_async_v4(uint32_t raddr, uint32_t rbar, uint32_t a, uint32_t b, uint32_t c,
                                            uint32_t d) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%2, %3, %4, %5}, [%1];" ::"r"(raddr),
               "r"(rbar), "r"(a), "r"(b), "r"(c), "r"(d)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t raddr) {   // release: prior reads of the buffer are done
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(raddr) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint32_t a, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAITC_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAITC_%=;\n\t}" ::"r"(a),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t mbar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(mbar)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, uint64_t tmap, int c0, int c1, uint32_t mbar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(tmap), "r"(c0), "r"(c1), "r"(mbar)
      : "memory");
}
__device__ __forceinline__ void tma_load_4d(uint32_t dst, uint64_t tmap, int c0, int c1, int c2, int c3,
                                            uint32_t mbar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(dst),
      "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(mbar)
      : "memory");
}
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
__device__ __forceinline__ void prefetch_tmap(uint64_t tmap) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(tmap) : "memory");
}
__device__ __forceinline__ void mbar_arrive_cnt(uint32_t a, uint32_t n) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async16_zfill(uint32_t dst, const void* src, bool zero) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %2, 0;\n\t"
      "cp.async.cg.shared.global [%0], [%1], 16, p;\n\t}" ::"r"(dst),
      "l"(src), "r"((int)zero)
      : "memory");
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
  // bar.sync is .aligned: every warp arrives converged (the dependency / split-K spins that precede
  // these barriers are run by whole warps with warp-uniform exit conditions; synccheck-clean)
  __syncwarp();
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ int fdiv(const FastDiv& f, int x) {
  return (int)((__umulhi((uint32_t)x, f.mul) + (uint32_t)x) >> f.shift);
}
__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// completion signal: release-ordered add (orders this CTA's prior writes, observed through the
// preceding bar.sync, before the counter update) — no full membar / L1 invalidate
__device__ __forceinline__ void red_release_add(int* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int atom_acqrel_add(int* p, int v) {
  int old;
  asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
// programmatic dependent launch: let the next stage's grid launch now; wait for the previous one
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
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
// K-major SWIZZLE_128B (the TMA 128 B-swizzled tile): 8-row atoms of 1024 B (SBO), LBO unused (1);
// the start address advances by 32 B per MMA K step inside the 128 B row.
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
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
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t* v) {
  __syncwarp();   // tcgen05.ld is .sync.aligned
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr)
      : "memory");
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
// accumulator access for the epilogue: TMEM (tcgen05 paths) or the CUDA-core FP32 registers (ET_F32X)
template <int DT>
__device__ __forceinline__ void acc_ld16(uint32_t taddr, const float* sacc, int c0, uint32_t* v) {
  if constexpr (DT == ET_F32X) {
    if (c0 == 0) {
#pragma unroll
      for (int e = 0; e < 16; ++e) v[e] = __float_as_uint(sacc[e]);
    } else {
#pragma unroll
      for (int e = 0; e < 16; ++e) v[e] = __float_as_uint(sacc[16 + e]);
    }
  } else {
    tmem_ld16(taddr, v);
  }
}
template <int DT>
__device__ __forceinline__ void acc_wait() {
  if constexpr (DT != ET_F32X) tmem_ld_wait();
}

__device__ __forceinline__ float tf32_round(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// Global stores as asm without a "memory" clobber: the descriptor table is read through generic
// pointers, so a plain C++ store (or __stcg) makes the compiler re-load every descriptor field it
// needs after each store, and a generic load behind a generic store waits for that store -- one
// memory round trip per store. These stores cannot alias the descriptors; ordering against the
// completion signals (asm volatile with "memory") is kept because volatile asm is never reordered.
__device__ __forceinline__ void stg_f32(void* p, float v) { asm volatile("st.global.f32 [%0], %1;" ::"l"(p), "f"(v)); }
__device__ __forceinline__ void stg_b16(void* p, unsigned short v) { asm volatile("st.global.b16 [%0], %1;" ::"l"(p), "h"(v)); }
__device__ __forceinline__ void stg_v2(void* p, uint32_t a, uint32_t b) {
  asm volatile("st.global.v2.b32 [%0], {%1, %2};" ::"l"(p), "r"(a), "r"(b));
}
__device__ __forceinline__ void stg_v4(void* p, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.global.v4.b32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(a), "r"(b), "r"(c), "r"(d));
}
__device__ __forceinline__ void red_add_v4(void* p, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}
__device__ __forceinline__ void stg_zero4_cg(void* p) {
  asm volatile("st.global.cg.v4.b32 [%0], {%1, %1, %1, %1};" ::"l"(p), "r"(0));
}
__device__ __forceinline__ unsigned short bf16_bits(float x) {
  __nv_bfloat16 h = __float2bfloat16_rn(x);
  return *reinterpret_cast<unsigned short*>(&h);
}

// ------------------------------------------------------------------------------- element access
// 16-byte vectors: 4 fp32 or 8 bf16 channels. All views have 16 B-aligned pixels/channel offsets.
struct Vec8 {
  float v[8];
};

// storage rounding: TF32 mode keeps activations TF32-representable (Z14); FP32-SIMT stores exact fp32
__device__ __forceinline__ float rnd(float x, int dtype) { return dtype == ET_F32 ? tf32_round(x) : x; }

__device__ __forceinline__ void load_vec(const View& vw, int dtype, int64_t pix, int c, float* out, int nv) {
  // nv = elements per 16 B (4 fp32 / 8 bf16); cache-global loads (other CTAs wrote these in this launch)
  if (dtype != ET_BF16) {
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
  if (dtype != ET_BF16) {
    stg_v4(reinterpret_cast<float*>(vw.ptr) + pix * vw.cstride + vw.coff + c, __float_as_uint(rnd(in[0], dtype)),
           __float_as_uint(rnd(in[1], dtype)), __float_as_uint(rnd(in[2], dtype)), __float_as_uint(rnd(in[3], dtype)));
  } else {
    uint4 a;
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&a);
#pragma unroll
    for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(in[2 * i], in[2 * i + 1]);
    stg_v4(reinterpret_cast<__nv_bfloat16*>(vw.ptr) + pix * vw.cstride + vw.coff + c, a.x, a.y, a.z, a.w);
  }
}

__device__ __forceinline__ float load_elem(const View& vw, int dtype, int64_t pix, int c) {
  if (dtype != ET_BF16) return __ldcg(reinterpret_cast<const float*>(vw.ptr) + pix * vw.cstride + vw.coff + c);
  const unsigned short* p = reinterpret_cast<const unsigned short*>(vw.ptr) + pix * vw.cstride + vw.coff + c;
  unsigned short u = __ldcg(p);
  return __uint_as_float(((uint32_t)u) << 16);
}
__device__ __forceinline__ void store_elem(const View& vw, int dtype, int64_t pix, int c, float x) {
  if (dtype != ET_BF16)
    stg_f32(reinterpret_cast<float*>(vw.ptr) + pix * vw.cstride + vw.coff + c, rnd(x, dtype));
  else
    stg_b16(reinterpret_cast<__nv_bfloat16*>(vw.ptr) + pix * vw.cstride + vw.coff + c, bf16_bits(x));
}

// ------------------------------------------------------------------------------ dependency waits
// Counters are never reset: every launch adds the same amounts, and launch number `ep` (the epoch,
// derived at kernel start from a 64-bit launch counter) turns the per-launch targets into absolute
// ones: wait until counter >= (ep + 1) * target. Both sides are taken mod 2^32 and compared
// wrap-safely ((int)(c - target) < 0): within one launch a counter is never more than one launch's
// increment away from its target, so the difference always fits an int, for any number of launches.
// A wait that exceeds ~4 s stores 1 into the error flag (host-mapped pinned memory: the host reads it
// without a copy; IOS_ERR_KERNEL from the next ios_run / ios_run_host / ios_sync) and gives up.
__device__ __forceinline__ bool before(int c, uint32_t target) { return (int)((uint32_t)c - target) < 0; }
__device__ __forceinline__ void flag_error(int* err) {
  asm volatile("st.volatile.global.s32 [%0], %1;" ::"l"(err), "r"(1) : "memory");
}
// Called by a WHOLE warp: every lane polls the counter (one broadcast load per round) and the exit
// decision is lane 0's, shuffled, so the warp leaves converged (the named barriers that follow are
// .aligned).
__device__ __forceinline__ bool spin_until(const int* c, uint32_t target, int* err, long long t0, int lane) {
  bool done = !before(ld_acquire(c), target);
  if (!done && clock64() - t0 > (long long)8000000000LL) {   // ~4 s: deadlock guard -> IOS_ERR_KERNEL
    if (lane == 0) flag_error(err);
    done = true;
  }
  return __shfl_sync(0xffffffffu, done ? 1 : 0, 0) != 0;
}
#ifndef IOS_ROW_BANDS
__device__ __forceinline__ void wait_deps(const Problem& P, int* counters, int* err, uint32_t ep, int lane) {
  for (int d = 0; d < P.n_deps; ++d) {
    const int* c = counters + P.dep_idx[d];
    const uint32_t target = (ep + 1u) * (uint32_t)P.dep_target[d];
    const long long t0 = clock64();
    while (!spin_until(c, target, err, t0, lane)) __nanosleep(64);
  }
}
#define IOS_BAND_SIGNAL(band) \
  do {                        \
  } while (0)
#else
// Row-band dependencies (opt-in build: tools/build_variant.py bands -DIOS_ROW_BANDS).
// Measured (1 B200, interleaved): the Inception stem stage (three chained big-M convs, each 1.2 waves)
// 30.5 -> 26.5 us, other chain stages unchanged, but the extra wait / signal code cost 2-3 % on every
// other stage (Inception IOS schedule 0.517 -> 0.530 ms), so the default build leaves it out.
#define IOS_BAND_SIGNAL(band)                                                          \
  do {                                                                                 \
    if (P.band_ctr >= 0) red_release_add(counters + P.band_ctr + (band), 1);          \
  } while (0)
// g0..g1: the global input rows (n * H + h) this tile reads; a dependency in band mode waits only for
// the producer bands covering them, otherwise for the whole producer. Called by a
// whole warp: the lanes poll all needed counters (every dependency, every band) in parallel -- one
// round trip per polling round instead of one acquire per counter (measured: sequential acquires
// made band waits slower than whole-producer waits; relaxed polls + one fence.acq_rel were slower
// still).
static __device__ __noinline__ void wait_deps(const Problem& P, const DepBand* bands, int* counters, int* err, uint32_t ep,
                                       int lane, int g0, int g1) {
  int cb[6], lo[6], hi[6];
  uint32_t tg[6];
  const int nd = min(P.n_deps, 6);
#pragma unroll
  for (int d = 0; d < 6; ++d) {
    if (d >= nd) break;
    const DepBand* B = P.band_begin >= 0 ? bands + P.band_begin + d : nullptr;
    if (!B || B->mode == 0) {
      cb[d] = P.dep_idx[d];
      lo[d] = hi[d] = 0;
      tg[d] = (ep + 1u) * (uint32_t)P.dep_target[d];
      continue;
    }
    int b0, b1;
    if (B->mode == 2) {
      const int i0 = (g0 / B->H) / B->tN * B->tiles_h + (g0 % B->H) / B->tR;
      const int i1 = (g1 / B->H) / B->tN * B->tiles_h + (g1 % B->H) / B->tR;
      b0 = i0 * B->tiles_w;
      b1 = i1 * B->tiles_w + B->tiles_w - 1;
    } else {
      const int per_row = B->mode == 4 ? B->tiles_w : B->W;   // items per global row
      b0 = g0 * per_row / B->bsz;
      b1 = (g1 * per_row + per_row - 1) / B->bsz;
    }
    cb[d] = B->ctr;
    lo[d] = b0;
    hi[d] = min(b1, B->nbands - 1);
    tg[d] = (ep + 1u) * (uint32_t)B->target;
  }
  // flatten (dependency, band) pairs; lane i polls items i, i + 32, ... (acquire loads: a lane's
  // acquire plus the named barrier that follows orders the producers' writes for the whole CTA)
  int first[7];
  first[0] = 0;
#pragma unroll
  for (int d = 0; d < 6; ++d) first[d + 1] = first[d] + (d < nd ? hi[d] - lo[d] + 1 : 0);
  const int total = first[nd];
  const long long t0 = clock64();
  for (;;) {
    bool ok = true;
    for (int k = lane; k < total; k += 32) {
      int d = 0;
#pragma unroll
      for (int e = 1; e < 6; ++e) d += (e < nd && k >= first[e]) ? 1 : 0;
      ok &= !before(ld_acquire(counters + cb[d] + lo[d] + (k - first[d])), tg[d]);
    }
    if (__all_sync(0xffffffffu, ok)) break;
    const bool late = __shfl_sync(0xffffffffu, (clock64() - t0 > (long long)8000000000LL) ? 1 : 0, 0) != 0;
    if (late) {   // ~4 s deadlock guard -> IOS_ERR_KERNEL
      if (lane == 0) flag_error(err);
      break;
    }
    __nanosleep(64);
  }
}

// input rows (global g = n * H + h) read by output rows oh0..oh1 of images n0..n1 through a window of
// k rows, stride s, padding p over an input of height H
__device__ __forceinline__ void window_rows(int n0, int oh0, int n1, int oh1, int k, int s, int p, int H, int& g0,
                                            int& g1) {
  g0 = n0 * H + max(0, oh0 * s - p);
  g1 = n1 * H + min(H - 1, oh1 * s - p + k - 1);
}
// rows read by GEMM tile mt (non-swap: dense 128-pixel tiles or patch tiles; swap-AB: every row)
static __device__ __noinline__ void gemm_rows(const Problem& P, int Hin, int mt, int& g0, int& g1) {
  if (P.swap_ab) {
    g0 = 0;
    g1 = P.batch * Hin - 1;
    return;
  }
  const int k = P.fdw ? P.dk : P.kh, st = P.fdw ? P.ds : P.sh, pd = P.fdw ? P.dp : P.ph;
  int n0, n1, oh0, oh1;
  if (P.tt) {
    const int rr = fdiv(P.fd_tilw, mt);
    const int tnn = fdiv(P.fd_tilh, rr);
    const int th = rr - tnn * P.tiles_h;
    n0 = tnn * P.tN;
    n1 = min(P.batch, n0 + P.tN) - 1;
    oh0 = th * P.tR;
    oh1 = min(P.Ho, oh0 + P.tR) - 1;
  } else {
    const int hw = P.Ho * P.Wo;
    const int p0 = mt * kBM, p1 = min(P.M, p0 + kBM) - 1;
    n0 = p0 / hw;
    oh0 = (p0 - n0 * hw) / P.Wo;
    n1 = p1 / hw;
    oh1 = (p1 - n1 * hw) / P.Wo;
  }
  window_rows(n0, oh0, n1, oh1, k, st, pd, Hin, g0, g1);
}
// rows read by SIMT tile `tile` (items: pixels, or quads of dwq pixels along a row; global pools: all)
static __device__ __noinline__ void simt_rows(const Problem& P, int Hin, int tile, int& g0, int& g1) {
  const int i0 = tile * P.items_per_tile, i1 = min(i0 + P.items_per_tile, P.n_items) - 1;
  if (P.kind == PK_GAVGPOOL || i1 < i0) {
    g0 = 0;
    g1 = P.batch * Hin - 1;
    return;
  }
  int r0, r1;   // output global rows
  if (P.dwq) {
    const int wq = (P.Wo + P.dwq - 1) / P.dwq;
    r0 = i0 / wq;
    r1 = i1 / wq;
  } else {
    r0 = i0 / P.Wo;
    r1 = i1 / P.Wo;
  }
  window_rows(r0 / P.Ho, r0 % P.Ho, r1 / P.Ho, r1 % P.Ho, P.kh, P.sh, P.ph, Hin, g0, g1);
}
#endif  // IOS_ROW_BANDS

// split-K rendezvous: every split of an output tile arrives after its reductions, then waits for
// all `n` (the splits of one tile run on distinct, co-resident CTAs; a tile's splits only wait for
// tiles with higher indices, which the CTAs reach after finishing lower ones: no cycle)
__device__ __forceinline__ void split_rendezvous(int* ctr, int n, int* err, uint32_t ep, int lane) {
  if (lane == 0) atom_acqrel_add(ctr, 1);
  __syncwarp();
  const uint32_t target = (ep + 1u) * (uint32_t)n;
  const long long t0 = clock64();
  while (!spin_until(ctr, target, err, t0, lane)) __nanosleep(32);
}

// -------------------------------------------------------------------------------- SIMT tile body
// Memory-bound members. Items are (output pixel, 16 B channel vector); consecutive
// threads take consecutive vectors of one pixel (coalesced). Code size matters as much as ILP
// here: the whole stage kernel shares one instruction cache, so this body is one __noinline__
// function with short, register-resident loops (3-wide window rows: 3 loads in flight per row).
template <int DT>
__device__ __forceinline__ void ld16(const View& vw, int64_t pix, int c, float* out) {
  load_vec(vw, DT, pix, c, out, DT == ET_BF16 ? 8 : 4);
}

// Window ops with a square k x k window (k in {3, 5, 7}) and stride s in {1, 2}: each item is a
// quad of QW horizontally adjacent output pixels x one 16 B channel vector. Per window row the
// thread loads the (QW-1)*s + k input pixels the quad needs, all in flight at once, and reuses
// each for up to k taps x QW outputs (the generic path reloads every tap of every output).
// KIND 0: sepconv front half ReLU(sum_i w_i x_i) -> depthwise (weights tap-major [k*k][C] fp32);
// KIND 1: max pool (padding = -inf); KIND 2: avg pool (divisor per output as the generic path).
template <int DT>
constexpr int win_qw() { return DT == ET_BF16 ? 2 : 4; }

template <int DT, int K, int S, int KIND>
__device__ __noinline__ void win_tile(const Problem& P, const View* views, int tile, int tid, int nthr) {
  constexpr int NV = DT == ET_BF16 ? 8 : 4;
  constexpr int QW = win_qw<DT>();
  constexpr int SPAN = (QW - 1) * S + K;
  // descriptor fields and views by value (registers / local memory): no descriptor re-loads
  // behind this tile's global stores
  const View out = P.out;
  const View in = views[P.in_begin];
  const int nvec = out.C / NV;
  const int item0 = tile * P.items_per_tile;
  const int item1 = min(item0 + P.items_per_tile, P.n_items);
  const int total = (item1 - item0) * nvec;
  const int Ho = P.Ho, Wo = P.Wo, ph = P.ph, pw = P.pw, flags = P.flags;
  const int wq = (Wo + QW - 1) / QW;
  const int cs = in.C;
  const float* wd = reinterpret_cast<const float*>(P.wts);
  const int nin = KIND == 0 ? min(P.n_in, 8) : 1;
  View vin[KIND == 0 ? 8 : 1];
  float awv[KIND == 0 ? 8 : 1];
  if (KIND == 0) {
    const float* aw = reinterpret_cast<const float*>(P.add_w);
    for (int s = 0; s < nin; ++s) {
      vin[s] = views[P.in_begin + s];
      awv[s] = aw ? __ldg(aw + s) : 1.0f;
    }
  }
  const float neutral = KIND == 1 ? -INFINITY : 0.f;
  for (int idx = tid; idx < total; idx += nthr) {
    const int qi = idx / nvec;
    const int c = (idx - qi * nvec) * NV;
    const int q = item0 + qi;
    const int row = q / wq;                       // n * Ho + oh
    const int ow0 = (q - row * wq) * QW;
    const int n = row / Ho, oh = row - n * Ho;
    const int hs = oh * S - ph, ws = ow0 * S - pw;
    float acc[QW][NV];
#pragma unroll
    for (int u = 0; u < QW; ++u)
#pragma unroll
      for (int e = 0; e < NV; ++e) acc[u][e] = neutral;
    // rows fully unrolled with a validity predicate (no early `continue`), so the loads of
    // several window rows can be in flight together
#pragma unroll
    for (int i = 0; i < K; ++i) {
      const int ih = hs + i;
      const bool rok = (unsigned)ih < (unsigned)in.H;
      const int64_t rowpix = ((int64_t)n * in.H + (rok ? ih : 0)) * in.W + ws;
      float xr[SPAN][NV];
      if (KIND == 0 && nin > 1) {
#pragma unroll
        for (int t = 0; t < SPAN; ++t)
#pragma unroll
          for (int e = 0; e < NV; ++e) xr[t][e] = 0.f;
        #pragma unroll 1
        for (int s = 0; s < nin; ++s) {
          const View& vs = vin[s];
          const float w = awv[s];
#pragma unroll
          for (int t = 0; t < SPAN; ++t) {
            if (rok && (unsigned)(ws + t) < (unsigned)in.W) {
              float x[NV];
              ld16<DT>(vs, rowpix + t, c, x);
#pragma unroll
              for (int e = 0; e < NV; ++e) xr[t][e] = fmaf(w, x[e], xr[t][e]);
            }
          }
        }
      } else {
#pragma unroll
        for (int t = 0; t < SPAN; ++t) {
          if (rok && (unsigned)(ws + t) < (unsigned)in.W) {
            ld16<DT>(in, rowpix + t, c, xr[t]);
          } else {
#pragma unroll
            for (int e = 0; e < NV; ++e) xr[t][e] = neutral;
          }
        }
      }
      if (KIND == 0) {
#pragma unroll
        for (int t = 0; t < SPAN; ++t)
#pragma unroll
          for (int e = 0; e < NV; ++e) xr[t][e] = fmaxf(xr[t][e], 0.f);   // padding stays 0
#pragma unroll
        for (int j = 0; j < K; ++j) {
          float w[NV];
          const float4* wp = reinterpret_cast<const float4*>(wd + (int64_t)(i * K + j) * cs + c);
#pragma unroll
          for (int h = 0; h < NV / 4; ++h) {
            const float4 v = __ldg(wp + h);
            w[4 * h] = v.x; w[4 * h + 1] = v.y; w[4 * h + 2] = v.z; w[4 * h + 3] = v.w;
          }
#pragma unroll
          for (int u = 0; u < QW; ++u)
#pragma unroll
            for (int e = 0; e < NV; ++e) acc[u][e] = fmaf(w[e], xr[u * S + j][e], acc[u][e]);
        }
      } else {
#pragma unroll
        for (int j = 0; j < K; ++j)
#pragma unroll
          for (int u = 0; u < QW; ++u)
#pragma unroll
            for (int e = 0; e < NV; ++e)
              acc[u][e] = KIND == 1 ? fmaxf(acc[u][e], xr[u * S + j][e]) : acc[u][e] + xr[u * S + j][e];
      }
    }
#pragma unroll
    for (int u = 0; u < QW; ++u) {
      const int ow = ow0 + u;
      if (ow >= Wo) break;
      if (KIND == 2) {
        const int wsu = ws + u * S;
        const int he = min(hs + K, in.H + ph), we = min(wsu + K, in.W + pw);
        int div;
        if (flags & 8) div = (he - hs) * (we - wsu);
        else div = (min(he, in.H) - max(hs, 0)) * (min(we, in.W) - max(wsu, 0));
        const float inv = 1.0f / (float)div;
#pragma unroll
        for (int e = 0; e < NV; ++e) acc[u][e] *= inv;
      }
      store_vec(out, DT, (int64_t)row * Wo + ow, c, acc[u]);
    }
  }
}

template <int DT>
__device__ __forceinline__ bool win_dispatch(const Problem& P, const View* views, int tile, int tid, int nthr) {
  const int k = P.kh, s = P.sh;
  if (P.kind == PK_DWCONV) {
    if (k == 3 && s == 1) win_tile<DT, 3, 1, 0>(P, views, tile, tid, nthr);
    else if (k == 3 && s == 2) win_tile<DT, 3, 2, 0>(P, views, tile, tid, nthr);
    else if (k == 5 && s == 1) win_tile<DT, 5, 1, 0>(P, views, tile, tid, nthr);
    else if (k == 5 && s == 2) win_tile<DT, 5, 2, 0>(P, views, tile, tid, nthr);
    else if (k == 7 && s == 1) win_tile<DT, 7, 1, 0>(P, views, tile, tid, nthr);
    else if (k == 7 && s == 2) win_tile<DT, 7, 2, 0>(P, views, tile, tid, nthr);
    else return false;
  } else if (P.kind == PK_MAXPOOL && k == 3) {
    if (s == 1) win_tile<DT, 3, 1, 1>(P, views, tile, tid, nthr);
    else if (s == 2) win_tile<DT, 3, 2, 1>(P, views, tile, tid, nthr);
    else return false;
  } else if (P.kind == PK_AVGPOOL && k == 3) {
    if (s == 1) win_tile<DT, 3, 1, 2>(P, views, tile, tid, nthr);
    else if (s == 2) win_tile<DT, 3, 2, 2>(P, views, tile, tid, nthr);
    else return false;
  } else {
    return false;
  }
  return true;
}

// Fused Relu-SepConv A operand. One 128 B channel chunk of a patch M tile (tN
// images x tR rows x tWt columns, tile row r = (nn*tR + i)*tWt + j, as the epilogue maps it): the
// producer warps compute ReLU(sum_i w_i x_i) -> k x k depthwise with the quad window walk of
// win_tile and store the values, rounded to the storage precision (Z14), straight into the UMMA
// SWIZZLE_NONE K-major layout [r/8][piece][r%8][16 B] the pointwise GEMM's MMAs read. The
// depthwise output never goes to HBM and the pointwise half needs no dependency round.
// Items = (quad of QW adjacent patch columns) x (16 B piece); 8 consecutive threads take the 8
// pieces of one quad (coalesced 128 B loads of one pixel's chunk).
template <int DT, int K, int S>
__device__ __noinline__ void fdw_chunk(const Problem& P, const View* views, uint32_t dst, int chunk, int tn0,
                                       int toh0, int tow0, int ptid) {
  constexpr int NV = DT == ET_BF16 ? 8 : 4;
  constexpr int QW = win_qw<DT>();
  constexpr int SPAN = (QW - 1) * S + K;
  const int tR = P.tR, tWt = P.tWt, nb = P.batch, Ho = P.Ho;
  const int qwn = (tWt + QW - 1) / QW;
  const int items = P.tN * tR * qwn * 8;
  const View in = views[P.in_begin];
  const int cs = in.C, inH = in.H, inW = in.W, dp = P.dp;
  const float* wd = reinterpret_cast<const float*>(P.dww);
  const int nin = min(P.n_in, 8);
  View vin[8];
  float awv[8];
  {
    const float* aw = reinterpret_cast<const float*>(P.add_w);
    for (int s = 0; s < nin; ++s) {
      vin[s] = views[P.in_begin + s];
      awv[s] = aw ? __ldg(aw + s) : 1.0f;
    }
  }
  for (int idx = ptid; idx < items; idx += 128) {
    const int piece = idx & 7;
    const int q = idx >> 3;
    const int rowi = q / qwn;                  // nn * tR + i
    const int qj = q - rowi * qwn;
    const int nn = rowi / tR, i0 = rowi - nn * tR;
    const int n = tn0 + nn, oh = toh0 + i0, ow0 = tow0 + qj * QW;
    const int c = chunk * (8 * NV) + piece * NV;
    float acc[QW][NV];
#pragma unroll
    for (int u = 0; u < QW; ++u)
#pragma unroll
      for (int e = 0; e < NV; ++e) acc[u][e] = 0.f;
    if (n < nb && oh < Ho && c < cs) {
      const int hs = oh * S - dp, ws = ow0 * S - dp;
#pragma unroll
      for (int i = 0; i < K; ++i) {
        const int ih = hs + i;
        const bool rok = (unsigned)ih < (unsigned)inH;
        const int64_t rowpix = ((int64_t)n * inH + (rok ? ih : 0)) * inW + ws;
        float xr[SPAN][NV];
        if (nin > 1) {
#pragma unroll
          for (int t = 0; t < SPAN; ++t)
#pragma unroll
            for (int e = 0; e < NV; ++e) xr[t][e] = 0.f;
          #pragma unroll 1
          for (int s = 0; s < nin; ++s) {
            const View& vs = vin[s];
            const float w = awv[s];
#pragma unroll
            for (int t = 0; t < SPAN; ++t) {
              if (rok && (unsigned)(ws + t) < (unsigned)inW) {
                float x[NV];
                ld16<DT>(vs, rowpix + t, c, x);
#pragma unroll
                for (int e = 0; e < NV; ++e) xr[t][e] = fmaf(w, x[e], xr[t][e]);
              }
            }
          }
        } else {
          const float w = awv[0];
#pragma unroll
          for (int t = 0; t < SPAN; ++t) {
            if (rok && (unsigned)(ws + t) < (unsigned)inW) {
              ld16<DT>(in, rowpix + t, c, xr[t]);
#pragma unroll
              for (int e = 0; e < NV; ++e) xr[t][e] *= w;
            } else {
#pragma unroll
              for (int e = 0; e < NV; ++e) xr[t][e] = 0.f;
            }
          }
        }
#pragma unroll
        for (int t = 0; t < SPAN; ++t)
#pragma unroll
          for (int e = 0; e < NV; ++e) xr[t][e] = fmaxf(xr[t][e], 0.f);   // padding stays 0
#pragma unroll
        for (int j = 0; j < K; ++j) {
          float w[NV];
          const float4* wp = reinterpret_cast<const float4*>(wd + (int64_t)(i * K + j) * cs + c);
#pragma unroll
          for (int h = 0; h < NV / 4; ++h) {
            const float4 v = __ldg(wp + h);
            w[4 * h] = v.x; w[4 * h + 1] = v.y; w[4 * h + 2] = v.z; w[4 * h + 3] = v.w;
          }
#pragma unroll
          for (int u = 0; u < QW; ++u)
#pragma unroll
            for (int e = 0; e < NV; ++e) acc[u][e] = fmaf(w[e], xr[u * S + j][e], acc[u][e]);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < QW; ++u) {
      const int j = qj * QW + u;
      if (j >= tWt) break;
      const int r = rowi * tWt + j;
      const uint32_t a = dst + (uint32_t)(r >> 3) * 1024u + (uint32_t)(r & 7) * 16u + (uint32_t)piece * 128u;
      uint32_t w4[4];
      if (DT == ET_BF16) {
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          __nv_bfloat162 b2 = __floats2bfloat162_rn(acc[u][2 * h], acc[u][2 * h + 1]);
          w4[h] = *reinterpret_cast<uint32_t*>(&b2);
        }
      } else {
#pragma unroll
        for (int h = 0; h < 4; ++h) w4[h] = __float_as_uint(tf32_round(acc[u][h]));
      }
      asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(w4[0]), "r"(w4[1]), "r"(w4[2]), "r"(w4[3])
                   : "memory");
    }
  }
}

// Halo path of the fused Relu-SepConv (single input): the chunk's input window (hhs x hws pixels x
// 128 B, dense [row][col][128 B], padding already zeros) and depthwise weights ([k*k][elems] fp32) sit
// in shared memory; items as in fdw_chunk, every operand an ld.shared.v4.
template <int DT, int K, int S>
__device__ __noinline__ void fdw_halo(const Problem& P, uint32_t hbuf, uint32_t wbuf, uint32_t dst, int toh0, int ptid) {
  constexpr int NV = DT == ET_BF16 ? 8 : 4;
  constexpr int QW = win_qw<DT>();
  constexpr int SPAN = (QW - 1) * S + K;
  constexpr int ELEMS = 8 * NV;
  const int tR = P.tR, tWt = P.tWt, hws = P.hws, Ho = P.Ho;
  const int qwn = (tWt + QW - 1) / QW;
  const int items = tR * qwn * 8;
  const float* aw = reinterpret_cast<const float*>(P.add_w);
  const float w0 = aw ? __ldg(aw) : 1.0f;
  for (int idx = ptid; idx < items; idx += 128) {
    const int piece = idx & 7;
    const int q = idx >> 3;
    const int i0 = q / qwn;
    const int qj = q - i0 * qwn;
    float acc[QW][NV];
#pragma unroll
    for (int u = 0; u < QW; ++u)
#pragma unroll
      for (int e = 0; e < NV; ++e) acc[u][e] = 0.f;
    if (toh0 + i0 < Ho) {
#pragma unroll
      for (int i = 0; i < K; ++i) {
        const uint32_t hrow = hbuf + (uint32_t)(((i0 * S + i) * hws + qj * QW * S) * 128 + piece * 16);
        float xr[SPAN][NV];
#pragma unroll
        for (int t = 0; t < SPAN; ++t) {
          uint32_t w[4];
          asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3])
                       : "r"(hrow + t * 128));
          if (DT == ET_BF16) {
#pragma unroll
            for (int h = 0; h < 4; ++h) {
              xr[t][2 * h] = __uint_as_float(w[h] << 16);
              xr[t][2 * h + 1] = __uint_as_float(w[h] & 0xffff0000u);
            }
          } else {
#pragma unroll
            for (int h = 0; h < 4; ++h) xr[t][h] = __uint_as_float(w[h]);
          }
#pragma unroll
          for (int e = 0; e < NV; ++e) xr[t][e] = fmaxf(xr[t][e] * w0, 0.f);
        }
#pragma unroll
        for (int j = 0; j < K; ++j) {
          float wv[NV];
#pragma unroll
          for (int h = 0; h < NV / 4; ++h) {
            uint32_t w[4];
            asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3])
                         : "r"(wbuf + (uint32_t)(((i * K + j) * ELEMS + piece * NV + 4 * h) * 4)));
#pragma unroll
            for (int e = 0; e < 4; ++e) wv[4 * h + e] = __uint_as_float(w[e]);
          }
#pragma unroll
          for (int u = 0; u < QW; ++u)
#pragma unroll
            for (int e = 0; e < NV; ++e) acc[u][e] = fmaf(wv[e], xr[u * S + j][e], acc[u][e]);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < QW; ++u) {
      const int j = qj * QW + u;
      if (j >= tWt) break;
      const int r = i0 * tWt + j;
      const uint32_t a = dst + (uint32_t)(r >> 3) * 1024u + (uint32_t)(r & 7) * 16u + (uint32_t)piece * 128u;
      uint32_t w4[4];
      if (DT == ET_BF16) {
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          __nv_bfloat162 b2 = __floats2bfloat162_rn(acc[u][2 * h], acc[u][2 * h + 1]);
          w4[h] = *reinterpret_cast<uint32_t*>(&b2);
        }
      } else {
#pragma unroll
        for (int h = 0; h < 4; ++h) w4[h] = __float_as_uint(tf32_round(acc[u][h]));
      }
      asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(w4[0]), "r"(w4[1]), "r"(w4[2]), "r"(w4[3])
                   : "memory");
    }
  }
}

template <int DT>
__device__ __forceinline__ void fdw_halo_dispatch(const Problem& P, uint32_t hbuf, uint32_t wbuf, uint32_t dst, int toh0,
                                                  int ptid) {
  const int k = P.dk, s = P.ds;
  if (k == 3 && s == 1) fdw_halo<DT, 3, 1>(P, hbuf, wbuf, dst, toh0, ptid);
  else if (k == 3 && s == 2) fdw_halo<DT, 3, 2>(P, hbuf, wbuf, dst, toh0, ptid);
  else if (k == 5 && s == 1) fdw_halo<DT, 5, 1>(P, hbuf, wbuf, dst, toh0, ptid);
  else if (k == 5 && s == 2) fdw_halo<DT, 5, 2>(P, hbuf, wbuf, dst, toh0, ptid);
  else if (k == 7 && s == 1) fdw_halo<DT, 7, 1>(P, hbuf, wbuf, dst, toh0, ptid);
  else fdw_halo<DT, 7, 2>(P, hbuf, wbuf, dst, toh0, ptid);
}

template <int DT>
__device__ __forceinline__ void fdw_dispatch(const Problem& P, const View* views, uint32_t dst, int chunk, int tn0,
                                             int toh0, int tow0, int ptid) {
  const int k = P.dk, s = P.ds;
  if (k == 3 && s == 1) fdw_chunk<DT, 3, 1>(P, views, dst, chunk, tn0, toh0, tow0, ptid);
  else if (k == 3 && s == 2) fdw_chunk<DT, 3, 2>(P, views, dst, chunk, tn0, toh0, tow0, ptid);
  else if (k == 5 && s == 1) fdw_chunk<DT, 5, 1>(P, views, dst, chunk, tn0, toh0, tow0, ptid);
  else if (k == 5 && s == 2) fdw_chunk<DT, 5, 2>(P, views, dst, chunk, tn0, toh0, tow0, ptid);
  else if (k == 7 && s == 1) fdw_chunk<DT, 7, 1>(P, views, dst, chunk, tn0, toh0, tow0, ptid);
  else fdw_chunk<DT, 7, 2>(P, views, dst, chunk, tn0, toh0, tow0, ptid);   // planner: k in {3,5,7}, s in {1,2}
}

template <int DT>
__device__ __noinline__ void simt_tile(const Problem& P, const View* views, int tile, int tid, int nthr) {
  constexpr int NV = DT == ET_BF16 ? 8 : 4;
  const View& out = P.out;
  const int nvec = out.C / NV;
  const int item0 = tile * P.items_per_tile;
  const int item1 = min(item0 + P.items_per_tile, P.n_items);
  if (P.dwq) {
    win_dispatch<DT>(P, views, tile, tid, nthr);   // the planner set dwq only for supported shapes
    return;
  }
  if (P.kind == PK_GAVGPOOL) {
    // 4 (image, channel vector) items per warp (items_per_tile / 4 warps: 4 on epilogue warps,
    // 9 when the stage runs SIMT on every warp): lane = (pixel phase p, item il); 8 pixel phases
    // per item, 8 loads in flight per lane, shuffle-reduced over the phases
    if (tid >= P.items_per_tile * 8) return;
    const View& in = views[P.in_begin];
    const int hw = in.H * in.W;
    const float inv = 1.0f / (float)hw;
    const bool relu = (P.flags & 2) != 0;
    const int lane = tid & 31, il = lane & 3, p = lane >> 2;
    const int idx = item0 + (tid >> 5) * 4 + il;
    const bool ok = idx < item1;
    const int n = ok ? idx / nvec : 0, v = ok ? idx - (idx / nvec) * nvec : 0;
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (ok) {
      for (int p0 = p; p0 < hw; p0 += 64) {
        float x[8][8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (p0 + 8 * u < hw) ld16<DT>(in, (int64_t)n * hw + p0 + 8 * u, v * NV, x[u]);
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (p0 + 8 * u < hw) {
#pragma unroll
            for (int e = 0; e < NV; ++e) acc[e] += relu ? fmaxf(x[u][e], 0.f) : x[u][e];
          }
      }
    }
#pragma unroll
    for (int e = 0; e < NV; ++e) {
      acc[e] += __shfl_xor_sync(0xffffffffu, acc[e], 4);
      acc[e] += __shfl_xor_sync(0xffffffffu, acc[e], 8);
      acc[e] += __shfl_xor_sync(0xffffffffu, acc[e], 16);
      acc[e] *= inv;
    }
    if (ok && p == 0) store_vec(out, DT, n, v * NV, acc);
    return;
  }
  const int total = (item1 - item0) * nvec;
  if (P.kind == PK_ADD && P.n_in <= 8) {
    // n-ary weighted add: inputs and weights by value (no descriptor re-loads behind the stores),
    // all inputs of an item loaded before the sum
    const View o = out;
    const int nin = P.n_in;
    View vin[8];
    float awv[8];
    const float* aw = reinterpret_cast<const float*>(P.add_w);
    for (int i = 0; i < nin; ++i) {
      vin[i] = views[P.in_begin + i];
      awv[i] = aw ? __ldg(aw + i) : 1.0f;
    }
    for (int idx = tid; idx < total; idx += nthr) {
      const int pix = item0 + idx / nvec;
      const int c = (idx % nvec) * NV;
      float x[8][8];
#pragma unroll
      for (int i = 0; i < 8; ++i)
        if (i < nin) ld16<DT>(vin[i], pix, c, x[i]);
      float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
      for (int i = 0; i < 8; ++i)
        if (i < nin) {
#pragma unroll
          for (int e = 0; e < NV; ++e) acc[e] = fmaf(awv[i], x[i][e], acc[e]);
        }
      store_vec(o, DT, pix, c, acc);
    }
    return;
  }
  const int HoWo = P.Ho * P.Wo;
  const float* aw = reinterpret_cast<const float*>(P.add_w);
  for (int idx = tid; idx < total; idx += nthr) {
    const int pix = item0 + idx / nvec;       // output pixel (n, oh, ow)
    const int c = (idx % nvec) * NV;
    const int n = pix / HoWo;
    const int rem = pix - n * HoWo;
    const int oh = rem / P.Wo, ow = rem - (rem / P.Wo) * P.Wo;
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (P.kind == PK_ADD) {
      for (int i = 0; i < P.n_in; ++i) {
        float x[8];
        ld16<DT>(views[P.in_begin + i], pix, c, x);
        const float w = aw ? aw[i] : 1.0f;
#pragma unroll
        for (int e = 0; e < NV; ++e) acc[e] = fmaf(w, x[e], acc[e]);
      }
    } else if (P.kind == PK_MAXPOOL || P.kind == PK_AVGPOOL || P.kind == PK_DWCONV) {
      // window rows; three taps of a row are loaded before use
      const View& in = views[P.in_begin];
      const bool is_max = P.kind == PK_MAXPOOL, is_dw = P.kind == PK_DWCONV;
      if (is_max) {
#pragma unroll
        for (int e = 0; e < NV; ++e) acc[e] = -INFINITY;
      }
      const float* wd = reinterpret_cast<const float*>(P.wts);
      const int hs = oh * P.sh - P.ph, ws = ow * P.sw - P.pw;
      const int nin = is_dw ? P.n_in : 1;
      for (int i = 0; i < P.kh; ++i) {
        const int ih = hs + i;
        if (ih < 0 || ih >= in.H) continue;
        const int64_t rowpix = ((int64_t)n * in.H + ih) * in.W;
        for (int j0 = 0; j0 < P.kw; j0 += 3) {
          float a0[8] = {0, 0, 0, 0, 0, 0, 0, 0}, a1[8] = {0, 0, 0, 0, 0, 0, 0, 0}, a2[8] = {0, 0, 0, 0, 0, 0, 0, 0};
          const int iw = ws + j0;
          const bool v0 = iw >= 0 && iw < in.W;
          const bool v1 = j0 + 1 < P.kw && iw + 1 >= 0 && iw + 1 < in.W;
          const bool v2 = j0 + 2 < P.kw && iw + 2 >= 0 && iw + 2 < in.W;
          for (int s = 0; s < nin; ++s) {     // sepconv: weighted sum of its inputs
            const View& vs = views[P.in_begin + s];
            const float w = (is_dw && aw) ? aw[s] : 1.0f;
            float x0[8], x1[8], x2[8];
            if (v0) ld16<DT>(vs, rowpix + iw, c, x0);
            if (v1) ld16<DT>(vs, rowpix + iw + 1, c, x1);
            if (v2) ld16<DT>(vs, rowpix + iw + 2, c, x2);
#pragma unroll
            for (int e = 0; e < NV; ++e) {
              if (v0) a0[e] = fmaf(w, x0[e], a0[e]);
              if (v1) a1[e] = fmaf(w, x1[e], a1[e]);
              if (v2) a2[e] = fmaf(w, x2[e], a2[e]);
            }
          }
          if (is_dw) {
            const int tap = i * P.kw + j0, cs = in.C;   // weights tap-major [kh*kw][C]
#pragma unroll
            for (int e = 0; e < NV; ++e) {
              const float* we = wd + (int64_t)tap * cs + c + e;
              if (v0) acc[e] = fmaf(__ldg(we), fmaxf(a0[e], 0.f), acc[e]);
              if (v1) acc[e] = fmaf(__ldg(we + cs), fmaxf(a1[e], 0.f), acc[e]);
              if (v2) acc[e] = fmaf(__ldg(we + 2 * cs), fmaxf(a2[e], 0.f), acc[e]);
            }
          } else {
#pragma unroll
            for (int e = 0; e < NV; ++e) {
              if (v0) acc[e] = is_max ? fmaxf(acc[e], a0[e]) : acc[e] + a0[e];
              if (v1) acc[e] = is_max ? fmaxf(acc[e], a1[e]) : acc[e] + a1[e];
              if (v2) acc[e] = is_max ? fmaxf(acc[e], a2[e]) : acc[e] + a2[e];
            }
          }
        }
      }
      if (P.kind == PK_AVGPOOL) {
        // divisor: window clipped to the padded input (include pad) or to the input (exclude pad)
        const int he = min(hs + P.kh, in.H + P.ph), we = min(ws + P.kw, in.W + P.pw);
        int div;
        if (P.flags & 8) div = (he - hs) * (we - ws);
        else div = (min(he, in.H) - max(hs, 0)) * (min(we, in.W) - max(ws, 0));
        const float inv = 1.0f / (float)div;
#pragma unroll
        for (int e = 0; e < NV; ++e) acc[e] *= inv;
      }
    } else {
      // PK_COPY: concat gather, element-wise (inputs may have non-vector channel counts)
      for (int e = 0; e < NV; ++e) {
        int ch = c + e, off = 0;
        for (int i = 0; i < P.n_in; ++i) {
          const View& vi = views[P.in_begin + i];
          if (ch < off + vi.Cl) {
            acc[e] = load_elem(vi, DT, pix, ch - off);
            break;
          }
          off += vi.Cl;
        }
      }
    }
    store_vec(out, DT, pix, c, acc);
  }
}

// --------------------------------------------------------------------------------- the kernel
struct Ring {          // smem ring iterator (slot, phase); n = slots this launch (StageDesc.ring_slots)
  int slot = 0;
  uint32_t phase = 0;
  int n = kStages;
  __device__ __forceinline__ void advance(int n) {
    for (int i = 0; i < n; ++i) next();
  }
  __device__ __forceinline__ void next() {
    if (++slot == n) {
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

// (split, m tile, n tile, K chunk range) of GEMM tile `local` of problem P
struct TileCoord {
  int s, mt, nt, c0, c1;
};
__device__ __forceinline__ TileCoord tile_coord(const Problem& P, int local) {
  TileCoord tc;
  const int rest = fdiv(P.fd_split, local);
  tc.s = local - rest * P.split;
  tc.mt = fdiv(P.fd_ntn, rest);
  tc.nt = rest - tc.mt * P.n_tiles_n;
  tc.c0 = tc.s * P.chunks_per_split;
  tc.c1 = min(tc.c0 + P.chunks_per_split, P.k_chunks);
  return tc;
}

// SD: the descriptor table fits the smem copy (the host picks the instantiation). The pointers are
// then derived from the shared array, so descriptor reads compile to shared loads, which do not
// wait behind outstanding global stores the way generic loads do.
template <int DT, bool SD, int FEAT>
__global__ void __launch_bounds__(kThreads, 1) ios_stage_kernel(const StageDesc sd) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // align by pointer arithmetic on the shared array (an integer round trip would make every
  // derived pointer generic: generic loads wait behind outstanding global stores)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  // ring slot s: A region (16 KB) at smem + s * slot_bytes, B region right after it
  const int slot_bytes = sd.slot_bytes;
  auto slotA = [&](int s) { return smem + s * slot_bytes; };
  auto slotB = [&](int s) { return smem + s * slot_bytes + kAStageBytes; };
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kRingBytes);
  uint64_t* full = bars;                                    // [kMaxSlots]
  uint64_t* empty = bars + kMaxSlots;                       // [kMaxSlots]
  uint64_t* tfull = bars + 2 * kMaxSlots;                   // [2]
  uint64_t* tempty = bars + 2 * kMaxSlots + 2;              // [2]
  uint64_t* hbar = bars + 2 * kMaxSlots + 4;                // [2] halo + depthwise weights landed (halo path)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kMaxSlots + 6);
  int* flag = reinterpret_cast<int*>(tmem_slot + 1);
  // cluster split-K (F_CSK): rfull = this CTA's receive buffer holds every peer's partial rows;
  // sempty[k] = the CTA of cluster rank k has consumed what this CTA last pushed to it
  uint64_t* rfull = bars + 2 * kMaxSlots + 7;                 // [1]
  uint64_t* sempty = bars + 2 * kMaxSlots + 8;                // [kClusterCtas]
  constexpr bool kCsk = (FEAT & F_CSK) != 0;
  const bool csk_launch = kCsk && sd.cluster > 1;
  float* sbias_all = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(bars) + kBarBytes);  // 2 x kMaxBN
  uint8_t* sdesc = reinterpret_cast<uint8_t*>(bars) + kBarBytes + kBiasBytes;           // kDescBytes
  uint8_t* sepi = sdesc + kDescBytes;                                                     // kEpiBytes: 4 x 4 KB
  __shared__ int sm_tile_begin[kMaxProblems];

  // The descriptor table is copied into shared memory once, so every role decodes its tiles from
  // smem instead of a chain of dependent global loads.
  constexpr bool desc_in_smem = SD;
  const uint8_t* dbase = SD ? sdesc : reinterpret_cast<const uint8_t*>(sd.problems);
  const Problem* probs = reinterpret_cast<const Problem*>(dbase);
  const View* views = reinterpret_cast<const View*>(dbase + sd.views_off);
  const Segment* segs = reinterpret_cast<const Segment*>(dbase + sd.segs_off);
#ifdef IOS_ROW_BANDS
  const DepBand* bands = reinterpret_cast<const DepBand*>(dbase + sd.bands_off);
#endif
  int* counters = reinterpret_cast<int*>(sd.counters);
  int* err = reinterpret_cast<int*>(sd.err);
  // optional per-CTA timeline (ns, %globaltimer) for tools/trace_stage.py; slots: 0 entry, 1 prologue
  // done, 2 first GEMM tile A issued, 3 producer done, 4 MMA done, 5 first accumulator ready,
  // 6 epilogue/SIMT done, 7 teardown, 8 exit
  // (only in the F_TRACE instantiation: the stamps cost registers and code in every hot loop)
  constexpr bool kTrace = (FEAT & F_TRACE) != 0;
  uint64_t* trace = kTrace && sd.trace ? reinterpret_cast<uint64_t*>(sd.trace) + blockIdx.x * 16 : nullptr;
  bool tfirst = kTrace && trace != nullptr;   // register flag: stamp only the first tile of each role
  // slot 0 = %globaltimer ns at entry (aligns CTAs); the other slots = SM cycles since entry + 1
  // (clock64 is a cheap register read; %globaltimer reads cost ~1 us each and distorted the timeline)
  const long long t_entry = kTrace ? clock64() : 0;
#define IOS_TRACE(slot)                                                        \
  do {                                                                         \
    if constexpr (kTrace)                                                      \
      if (trace) trace[(slot)] = (slot) == 0 ? gtimer() : (uint64_t)(clock64() - t_entry + 1); \
  } while (0)
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  if (tid == 0) IOS_TRACE(0);
  // Launch epoch: every CTA of a launch adds 1 to the plan's 64-bit launch counter (counters[0..1])
  // exactly once, before the launch triggers its dependents (launch_dependents below), so old / grid
  // is this launch's number for every CTA (it never wraps; the epoch itself is used mod 2^32). Every
  // CTA of an earlier launch of this plan added its 1 before that launch triggered ITS dependents,
  // so the value is final whenever this grid runs: the add is issued first thing, its L2 round trip
  // overlapping the descriptor copy and the barrier / TMEM set-up; the prologue barrier publishes it.
  unsigned long long ep_old = 0;
  if (sd.uses_counters && tid == 0) ep_old = atomicAdd(reinterpret_cast<unsigned long long*>(counters), 1ull);

  if (desc_in_smem) {
    const int4* src = reinterpret_cast<const int4*>(sd.problems);
    int4* dst = reinterpret_cast<int4*>(sdesc);
    for (int i = tid; i < (sd.blob_bytes + 15) / 16; i += kThreads) dst[i] = __ldg(src + i);
  }
  for (int i = tid; i < sd.n_problems; i += kThreads)
    sm_tile_begin[i] = reinterpret_cast<const Problem*>(sd.problems)[i].tile_begin;
  if (tid == 0) {
    for (int s = 0; s < sd.ring_slots; ++s) {
      mbar_init(smem_u32(&full[s]), kProducerWarps + 1);   // 4 producer warps + the expect_tx arrival
      mbar_init(smem_u32(&empty[s]), 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(smem_u32(&tfull[s]), 1);
      mbar_init(smem_u32(&tempty[s]), 128);
    }
    mbar_init(smem_u32(&hbar[0]), 1);
    mbar_init(smem_u32(&hbar[1]), 1);
    if (csk_launch) {
      mbar_init(smem_u32(rfull), 1);
      for (int k = 0; k < kClusterCtas; ++k) mbar_init(smem_u32(&sempty[k]), 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (sd.uses_counters) *flag = (int)(uint32_t)(ep_old / gridDim.x);
  }
  if (warp == kMmaWarp && sd.has_gemm && DT != ET_F32X) {
    __syncwarp();
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  // a cluster launch: every peer's barriers are initialised before anyone pushes into them (this
  // runs before the PDL wait, so it overlaps the previous stage's tail)
  if (csk_launch) {
    __syncwarp();
    cluster_sync_all();
  } else {
    __syncthreads();
  }
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // Weight prefetch into L2: weights are never written by earlier stages, so
  // before waiting for the previous grid every CTA asks L2 for its 1/grid share of each GEMM
  // member's packed weights; the stage's weight stream then overlaps the previous stage's tail.
#ifndef IOS_NO_PREFETCH
  if (warp == kMmaWarp && sd.has_gemm) {
    for (int q = lane; q < sd.n_problems; q += 32) {
      const Problem& P = probs[q];
      if (P.kind != PK_GEMM) continue;
#ifndef IOS_NO_TMAP_PREFETCH
      if (P.tmap_a) prefetch_tmap(P.tmap_a);   // descriptor fetch off the first TMA's critical path
#endif
      // (32-bit: packed weights of one GEMM are < 4 GB; a 64-bit division is a ~100-instruction call)
      const uint32_t total = (uint32_t)P.k_chunks * (uint32_t)P.Npad8 * kChunkBytes;
      const uint32_t share = ((total + gridDim.x - 1) / gridDim.x + 15) & ~15u;
      const uint32_t b0 = share * blockIdx.x, b1 = b0 + share < total ? b0 + share : total;
      for (uint32_t o = b0; o < b1; o += 32768)
        prefetch_l2(reinterpret_cast<const uint8_t*>(P.wts) + o, b1 - o < 32768 ? b1 - o : 32768);
    }
  }
#endif
  // Late PDL wait: no CTA-wide wait here. Each thread executes griddepcontrol.wait right before its
  // first access to data an earlier grid writes (activations; the split-K workspace): producers
  // after decoding their first tile (and its in-stage dependency wait: counters are this plan's own,
  // epoch-relative and monotonic, so they are safe to poll early), epilogue / SIMT threads before
  // their first tile's loads or stores; the MMA warp never touches global memory. Tile decode and
  // the code those paths first execute then overlap the previous stage's tail.
  bool pdl_done = false;
  auto lazy_pdl = [&]() {
    if (!pdl_done) {
      pdl_wait();
      pdl_done = true;
#ifdef IOS_TRACE_FINE
      if (tid == 0) IOS_TRACE(13);   // PDL wait returned
#endif
      if (sd.stamp && tid == 0) atomicMin(reinterpret_cast<unsigned long long*>(sd.stamp), (unsigned long long)gtimer());
    }
  };
  if (tid == 0) IOS_TRACE(11);
  pdl_launch_dependents();   // every CTA's epoch add is done (published by the prologue barrier)
  const uint32_t ep = sd.uses_counters ? (uint32_t)*flag : 0u;
  if (tid == 0) IOS_TRACE(1);

  if (!sd.has_gemm) {
    // ============================================================== SIMT-only stage: all warps
    int hint = 0;
    for (int t = blockIdx.x; t < sd.n_tiles; t += gridDim.x) {
      hint = find_problem(sm_tile_begin, sd.n_problems, t, hint);
      const Problem& P = probs[hint];
      lazy_pdl();
      if (warp == 0 && P.n_deps) {
#ifdef IOS_ROW_BANDS
        int g0, g1;
        simt_rows(P, views[P.in_begin].H, t - P.tile_begin, g0, g1);
        wait_deps(P, bands, counters, err, ep, lane, g0, g1);
#else
        wait_deps(P, counters, err, ep, lane);
#endif
      }
      named_bar(3, kThreads);
#ifndef IOS_NO_SIMT
      simt_tile<DT>(P, views, t - P.tile_begin, tid, kThreads);
#endif
      named_bar(3, kThreads);
      if (tid == 0 && P.signal) {
        red_release_add(counters + P.done_idx, 1);
        IOS_BAND_SIGNAL(t - P.tile_begin);
      }
    }
  } else if (warp < kProducerWarps) {
    // ============================================================== PRODUCER (A gather + B bulk)
    // Lean per-tile setup (fast divisions; per-row pixel offsets once per tile) and an incremental
    // im2col walk: each thread owns 2 pieces (16 B) x 4 rows of every 128 B K-chunk; a piece's
    // (tap row, tap col, channel) advance by one chunk per iteration without any division.
    const int ptid = tid;                       // 0..127
    const int rig = lane & 7;                   // row inside an 8-row core-matrix group
    const int pc0 = lane >> 3;                  // pieces pc0 and pc0 + 4 of each 128 B chunk row
    constexpr int ESZ = DT == ET_BF16 ? 2 : 4;
    constexpr int VEC = 16 / ESZ, ELEMS = kChunkBytes / ESZ;
    Ring ring;
    ring.n = sd.ring_slots;
    uint32_t hphase = 0;                        // halo barrier phase (fused Relu-SepConv, halo path)
    int hint = 0;
    for (int t = blockIdx.x; t < sd.n_tiles; t += gridDim.x) {
      hint = find_problem(sm_tile_begin, sd.n_problems, t, hint);
      const Problem& P = probs[hint];
      if (P.kind != PK_GEMM) continue;
      const int local = t - P.tile_begin;
      if (kCsk && local >= P.n_tiles) continue;   // cluster-alignment padding tile
      if (ptid == 0 && tfirst) IOS_TRACE(3);
      const TileCoord tc = tile_coord(P, local);
#ifdef IOS_TRACE_FINE
      if (ptid == 0 && tfirst) IOS_TRACE(14);   // tile decoded
#endif
      const int mt = tc.mt, nt = tc.nt, c0 = tc.c0, c1 = tc.c1;
      if (P.n_deps) {
        if (warp == 0) {
#ifdef IOS_ROW_BANDS
          int g0, g1;
          gemm_rows(P, views[P.in_begin].H, mt, g0, g1);
          wait_deps(P, bands, counters, err, ep, lane, g0, g1);
#else
          wait_deps(P, counters, err, ep, lane);
#endif
        }
        named_bar(1, 128);
      }
      lazy_pdl();
      if constexpr ((FEAT & F_FDW) != 0 && DT != ET_F32X) if (P.fdw) {
        // fused Relu-SepConv: depthwise computed into the A slot, pointwise weights by bulk copy
        const int rr = fdiv(P.fd_tilw, mt);
        const int tw = mt - rr * P.tiles_w;
        const int tnn = fdiv(P.fd_tilh, rr);
        const int tn0 = tnn * P.tN, toh0 = (rr - tnn * P.tiles_h) * P.tR, tow0 = tw * P.tWt;
        const uint8_t* wsrc = reinterpret_cast<const uint8_t*>(P.wts) + (int64_t)(nt * P.BN >> 3) * 1024;
        const int64_t wstep = (int64_t)(P.Npad8 >> 3) * 1024;
        const uint32_t bbytes = (uint32_t)min(P.BN, P.Npad8 - nt * P.BN) * kChunkBytes;
        if (P.hws) {
          // halo path: per chunk ONE 4D tensor TMA stages the tile's input window (padding = OOB
          // zeros) and one bulk copy the chunk's depthwise weights; the items are then computed
          // from shared memory. Double-buffered: chunk c+1's window is in flight while chunk c is
          // computed (slot 3's B region = 2 windows of 16 KB, its A region = 2 x 8 KB of weights).
          // (halo stages run 3 slots of 48 KB; the 4th slot's regions hold the windows / weights)
          const uint32_t hbuf0 = smem_u32(slotB(kStages - 1));
          const uint32_t wbuf0 = smem_u32(slotA(kStages - 1));
          const uint32_t hbytes = (uint32_t)(P.hws * P.hhs) * kChunkBytes;
          const uint32_t wbytes = (uint32_t)(P.dk * P.dk * kChunkBytes / ESZ) * 4u;
          const int ih0 = toh0 * P.ds - P.dp, iw0 = tow0 * P.ds - P.dp;
          auto issue = [&](int c, int b) {
            const uint32_t hb = smem_u32(&hbar[b]);
            mbar_arrive_expect_tx(hb, hbytes + wbytes);
            tma_load_4d(hbuf0 + b * (kHaloBytes / 2), P.tmap_a, c * ELEMS, iw0, ih0, tn0, hb);
            bulk_g2s(wbuf0 + b * (kHaloWBytes / 2), reinterpret_cast<const uint8_t*>(P.dwc) + (int64_t)c * wbytes, wbytes,
                     hb);
          };
          named_bar(1, 128);   // every producer thread is done with the previous tile's windows
          if (ptid == 0) issue(c0, 0);
          for (int c = c0; c < c1; ++c) {
            const int b = (c - c0) & 1;
            mbar_wait(smem_u32(&empty[ring.slot]), ring.phase ^ 1u);
            if (c > c0) named_bar(1, 128);   // chunk c-1 (buffer b^1) fully consumed
            if (ptid == 0) {
              const uint32_t fb = smem_u32(&full[ring.slot]);
              mbar_arrive_expect_tx(fb, bbytes);
              bulk_g2s(smem_u32(slotB(ring.slot)), wsrc + c * wstep, bbytes, fb);
              if (c + 1 < c1) issue(c + 1, b ^ 1);
            }
            mbar_wait(smem_u32(&hbar[b]), (hphase >> b) & 1u);
            hphase ^= 1u << b;
            fdw_halo_dispatch<DT>(P, hbuf0 + b * (kHaloBytes / 2), wbuf0 + b * (kHaloWBytes / 2),
                                  smem_u32(slotA(ring.slot)), toh0, ptid);
            fence_proxy_async();
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(&full[ring.slot]));
            ring.next();
          }
          if (ptid == 0 && tfirst) IOS_TRACE(12);
          tfirst = false;
          continue;
        }
        for (int c = c0; c < c1; ++c) {
          mbar_wait(smem_u32(&empty[ring.slot]), ring.phase ^ 1u);
          if (ptid == 0) {
            const uint32_t fb = smem_u32(&full[ring.slot]);
            mbar_arrive_expect_tx(fb, bbytes);
            bulk_g2s(smem_u32(slotB(ring.slot)), wsrc + c * wstep, bbytes, fb);
          }
          fdw_dispatch<DT>(P, views, smem_u32(slotA(ring.slot)), c, tn0, toh0, tow0, ptid);
          fence_proxy_async();
          __syncwarp();
          if (lane == 0) mbar_arrive(smem_u32(&full[ring.slot]));   // one arrival per producer warp
          ring.next();
        }
        if (ptid == 0 && tfirst) IOS_TRACE(12);
        tfirst = false;
        continue;
      }
      if (P.a_tma || P.tt) {
        // A is a plain [M, C] matrix (1x1, stride 1): ONE tensor TMA per chunk (128 rows x 128 B,
        // 128 B swizzle, rows past M / channels past C zero-filled) + one bulk copy for B, both
        // issued by one thread; warps 1-3 only keep their ring position in step.
        // Tap TMA (P.tt): chunk c = (tap, channel block); ONE 4D tensor TMA brings that tap's input
        // pixels of the tile's output patch (element strides = conv strides; padding and channels
        // past C are out-of-bounds zeros) in the same 128 B-swizzled [row][128 B] layout.
        if (warp == 0) {
          const uint64_t tmap = P.tmap_a;
          const bool swap = P.swap_ab != 0;
          // weights: BN rows of tile nt into the B slot, or (swap-AB) 128 rows of tile mt into A
          const int wrow0 = swap ? mt * kBM : nt * P.BN, wrows = swap ? kBM : P.BN;
          const uint8_t* wsrc = reinterpret_cast<const uint8_t*>(P.wts) + (int64_t)(wrow0 >> 3) * 1024;
          const int64_t wstep = (int64_t)(P.Npad8 >> 3) * 1024;
          const uint32_t bbytes = (uint32_t)min(wrows, P.Npad8 - wrow0) * kChunkBytes;
          const int woff = swap ? 0 : kAStageBytes, xoff = swap ? kAStageBytes : 0;   // region in a slot
          const int xrow0 = swap ? 0 : mt * kBM;
          // tap-TMA patch origin (input coordinates of tap (0, 0)) and box bytes
          int tn0 = 0, ih0 = 0, iw0 = 0;
          uint32_t xbytes = kAStageBytes;
          const int kblk = P.kblk, kwid = P.kw;
          if (P.tt) {
            const int rr = fdiv(P.fd_tilw, swap ? 0 : mt);
            const int tw = (swap ? 0 : mt) - rr * P.tiles_w;
            const int tnn = fdiv(P.fd_tilh, rr);
            const int th = rr - tnn * P.tiles_h;
            tn0 = tnn * P.tN;
            ih0 = th * P.tR * P.sh - P.ph;
            iw0 = tw * P.tWt * P.sw - P.pw;
            xbytes = (uint32_t)(P.tN * P.tR * P.tWt) * kChunkBytes;
          }
#ifdef IOS_TRACE_FINE
          if (lane == 0 && tfirst) IOS_TRACE(15);   // TMA geometry ready
#endif
          // tap-TMA chunk c = (tap (ti, tj), channel block cb): decoded once for c0, then stepped
          const bool is_tt = P.tt != 0;
          int cb = 0, ti = 0, tj = 0;
          if (is_tt) {
            const int tap = fdiv(P.fd_kblk, c0);
            cb = c0 - tap * kblk;
            ti = fdiv(P.fd_kw, tap);
            tj = tap - ti * kwid;
          }
          const uint8_t* wsrc_c = wsrc + c0 * wstep;
          for (int c = c0; c < c1; ++c) {
            mbar_wait(smem_u32(&empty[ring.slot]), ring.phase ^ 1u);
            if (lane == 0) {
              const uint32_t fb = smem_u32(&full[ring.slot]);
              mbar_arrive_expect_tx(fb, xbytes + bbytes);
              if (tfirst && c == c0) IOS_TRACE(9);
              if (is_tt)
                tma_load_4d(smem_u32(slotA(ring.slot) + xoff), tmap, cb * ELEMS, iw0 + tj, ih0 + ti, tn0, fb);
              else
                tma_load_2d(smem_u32(slotA(ring.slot) + xoff), tmap, c * ELEMS, xrow0, fb);
              if (tfirst && c == c0) IOS_TRACE(10);
              bulk_g2s(smem_u32(slotA(ring.slot) + woff), wsrc_c, bbytes, fb);
              mbar_arrive_cnt(fb, kProducerWarps);   // stands in for the 4 producer warps' arrivals
              if (tfirst && c - c0 < 2) IOS_TRACE(c == c0 ? 2 : 12);
            }
            wsrc_c += wstep;
            if (++cb == kblk) {
              cb = 0;
              if (++tj == kwid) {
                tj = 0;
                ++ti;
              }
            }
            __syncwarp();
            ring.next();
          }
          tfirst = false;
        } else {
          ring.advance(c1 - c0);
        }
        // keep the four producer warps in step across a TMA tile: letting warps 1-3 run ahead into
        // a following cp.async tile while warp 0 still issues this tile's chunks faults on the GPU
        // (observed with a 1x1 TMA tile followed by an independent gather tile in one stage)
        named_bar(1, 128);
        continue;
      }
      // implicit-im2col gather (cp.async) path: compiled into the F_GATHER instantiations only;
      // the host never hands a gather problem to a kernel without it (stage_features)
      if constexpr ((FEAT & F_GATHER) != 0) {
      // everything the chunk loop needs lives in registers: the cp.async asm statements clobber
      // "memory", which would otherwise force the descriptor fields to be re-read from smem
      const View in = views[P.in_begin];
      const int inC = in.C, inH = in.H, inW = in.W, cstride = in.cstride;
      const int kh = P.kh, kw = P.kw;
      const bool relu_pre = (P.flags & 2) != 0;
      const bool swap = P.swap_ab != 0;
      int roff[4], ih0[4], iw0[4];   // row pixel offset (may be negative: padding) and window origin
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int m = (swap ? 0 : mt * kBM) + (warp + 4 * j) * 8 + rig;
        const int n = fdiv(P.fd_howo, m);
        const int rem = m - n * (P.Ho * P.Wo);
        const int oh = fdiv(P.fd_wo, rem);
        const int ow = rem - oh * P.Wo;
        ih0[j] = oh * P.sh - P.ph;
        iw0[j] = ow * P.sw - P.pw;
        roff[j] = m < P.M ? (n * inH + ih0[j]) * inW + iw0[j] : INT_MIN;   // INT_MIN: row past M
      }
      // piece state at chunk c0: k = c0*ELEMS + pc*VEC = tap*C + ci, tap = ti*kw + tj
      int ti[2], tj[2], ci[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int k = c0 * ELEMS + (pc0 + 4 * h) * VEC;
        const int tap = fdiv(P.fd_cin, k);
        ci[h] = k - tap * inC;
        ti[h] = fdiv(P.fd_kw, tap);
        tj[h] = tap - ti[h] * kw;
      }
      // weights: BN rows of n tile nt (B slot), or with swap-AB 128 rows of channel tile mt (A slot);
      // the last tile may run past the packed rows: copy only those (the rest of the smem tile is
      // stale and only feeds accumulator rows/columns that no output segment covers)
      const int wrow0 = swap ? mt * kBM : nt * P.BN, wrows = swap ? kBM : P.BN;
      const uint8_t* wsrc = reinterpret_cast<const uint8_t*>(P.wts) + (int64_t)(wrow0 >> 3) * 1024;
      const int64_t wstep = (int64_t)(P.Npad8 >> 3) * 1024;
      const uint32_t bbytes = (uint32_t)min(wrows, P.Npad8 - wrow0) * kChunkBytes;
      const int woff = swap ? 0 : kAStageBytes, xoff = swap ? kAStageBytes : 0;   // region in a slot
      const char* ibase = reinterpret_cast<const char*>(in.ptr) + (int64_t)in.coff * ESZ;
      // pre-ReLU convs: the gather stays asynchronous; once a chunk's copies have landed, each thread
      // applies the ReLU in place to the 8 pieces it copied itself (visible to it after wait_group)
      auto relu_pieces = [&](int slot) {
        const uint32_t b0 = smem_u32(slotA(slot) + xoff) + rig * 16 + pc0 * 128;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (roff[j] == INT_MIN) continue;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const uint32_t a = b0 + (warp + 4 * j) * 1024 + h * 512;
            uint32_t w[4];
            asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]) : "r"(a));
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              if (ESZ == 4) {
                w[q] = __float_as_uint(fmaxf(__uint_as_float(w[q]), 0.f));
              } else {
                __nv_bfloat162 hb = *reinterpret_cast<__nv_bfloat162*>(&w[q]);
                hb = __hmax2(hb, __floats2bfloat162_rn(0.f, 0.f));
                w[q] = *reinterpret_cast<uint32_t*>(&hb);
              }
            }
            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3])
                         : "memory");
          }
        }
      };
      int pend[2] = {-1, -1};
      for (int c = c0; c < c1; ++c) {
        mbar_wait(smem_u32(&empty[ring.slot]), ring.phase ^ 1u);
        if (ptid == 0) {
          const uint32_t fb = smem_u32(&full[ring.slot]);
          mbar_arrive_expect_tx(fb, bbytes);
          bulk_g2s(smem_u32(slotA(ring.slot) + woff), wsrc + c * wstep, bbytes, fb);
        }
        const uint32_t a_st = smem_u32(slotA(ring.slot) + xoff) + rig * 16 + pc0 * 128;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const bool kvalid = ti[h] < kh;                            // k < K
          const int toff = (ti[h] * inW + tj[h]) * cstride + ci[h];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            if (roff[j] == INT_MIN) continue;                        // row past M: never stored
            const int ih = ih0[j] + ti[h], iw = iw0[j] + tj[h];
            const bool ok = kvalid && (unsigned)ih < (unsigned)inH && (unsigned)iw < (unsigned)inW;
            // padding taps / K tail: zero fill without reading (ignore-src)
            const char* src = ibase + ((int64_t)roff[j] * cstride + (ok ? toff : 0)) * ESZ;
            const uint32_t dst = a_st + (warp + 4 * j) * 1024 + h * 512;
            cp_async16_zfill(dst, ok ? src : ibase, !ok);
          }
          // advance this piece by one chunk (ELEMS elements of K)
          ci[h] += ELEMS;
          while (ci[h] >= inC) {
            ci[h] -= inC;
            if (++tj[h] == kw) {
              tj[h] = 0;
              ++ti[h];
            }
          }
        }
        cp_async_commit();
        if (ptid == 0 && tfirst && c - c0 < 3) IOS_TRACE(c == c0 ? 2 : 8 + c - c0);
        // arrive for the chunk issued two iterations ago (keeps up to 3 chunks of cp.async in flight)
        if (pend[0] >= 0) {
          cp_async_wait<2>();
          if (relu_pre) relu_pieces(pend[0]);
          fence_proxy_async();
          __syncwarp();
          if (lane == 0) mbar_arrive(smem_u32(&full[pend[0]]));   // one arrival per producer warp
        }
        pend[0] = pend[1];
        pend[1] = ring.slot;
        ring.next();
      }
      cp_async_wait<0>();
      if (relu_pre) {
        if (pend[0] >= 0) relu_pieces(pend[0]);
        if (pend[1] >= 0) relu_pieces(pend[1]);
      }
      if (ptid == 0 && tfirst) IOS_TRACE(12);
      tfirst = false;
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) {
        if (pend[0] >= 0) mbar_arrive(smem_u32(&full[pend[0]]));
        if (pend[1] >= 0) mbar_arrive(smem_u32(&full[pend[1]]));
      }
      }   // F_GATHER
    }
  } else if (warp == kMmaWarp) {
    // ============================================================== MMA ISSUER
    // The whole warp walks the tiles and waits on the barriers (warp-uniform control flow); one
    // elected lane issues tcgen05.mma / tcgen05.commit.
    if (sd.has_gemm && DT != ET_F32X) {
      Ring ring;
      ring.n = sd.ring_slots;
      int acc = 0;
      uint32_t acc_phase = 0;
      int hint = 0;
      for (int t = blockIdx.x; t < sd.n_tiles; t += gridDim.x) {
        hint = find_problem(sm_tile_begin, sd.n_problems, t, hint);
        const Problem& P = probs[hint];
        if (P.kind != PK_GEMM) continue;
        const int local = t - P.tile_begin;
        if (kCsk && local >= P.n_tiles) continue;   // cluster-alignment padding tile
        const int s = local - fdiv(P.fd_split, local) * P.split;
        const int c0 = s * P.chunks_per_split;
        const int c1 = min(c0 + P.chunks_per_split, P.k_chunks);
        const uint32_t idesc = umma_idesc(DT == ET_BF16, P.BN);
        // the activation operand is 128 B-swizzled when TMA loads it; swap-AB puts it in the B slot
        const bool act_tma = (P.a_tma != 0 || P.tt != 0) && !P.fdw;
        const bool a_sw128 = act_tma && !P.swap_ab;
        const bool b_sw128 = act_tma && P.swap_ab;
        mbar_wait(smem_u32(&tempty[acc]), acc_phase ^ 1u);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + (uint32_t)acc * kMaxBN;
        for (int c = c0; c < c1; ++c) {
          mbar_wait(smem_u32(&full[ring.slot]), ring.phase);
          tc_fence_after();
          const uint32_t a0 = smem_u32(slotA(ring.slot));
          const uint32_t b0 = smem_u32(slotB(ring.slot));
          __syncwarp();
          if (elect_one()) {
            // descriptor of the chunk's first 32 B of K; each next 32 B step moves the start address
            // field (address >> 4) by 2 (128 B-swizzled rows) or 16 (core-matrix layout, 256 B)
            const uint64_t ad = a_sw128 ? umma_desc_sw128(a0) : umma_desc(a0, 128, 1024);
            const uint64_t bd = b_sw128 ? umma_desc_sw128(b0) : umma_desc(b0, 128, 1024);
            const uint32_t astep = a_sw128 ? 2u : 16u, bstep = b_sw128 ? 2u : 16u;
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)   // 4 x 32 B of K per 128 B chunk
              umma<DT>(tmem_d, ad + kk * astep, bd + kk * bstep, idesc, (c > c0 || kk > 0) ? 1u : 0u);
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
    Ring ering;                                   // FP32-SIMT mode: the epilogue consumes the smem ring
    ering.n = sd.ring_slots;
    const int lane_base = (warp & 3) * 32;        // TMEM lanes this warp may access
    int acc = 0;
    uint32_t acc_phase = 0;
    // cluster split-K flow control (every epilogue warp keeps the same view): bit k of csk_sbits =
    // parity of sempty[k]'s completed phases; csk_rphase = parity of rfull's
    uint32_t csk_sbits = 0, csk_rphase = 0;
    int hint = 0;
    for (int t = blockIdx.x; t < sd.n_tiles; t += gridDim.x) {
      hint = find_problem(sm_tile_begin, sd.n_problems, t, hint);
      const Problem& P = probs[hint];
      if (kCsk && t - P.tile_begin >= P.n_tiles) continue;   // cluster-alignment padding tile
      if (P.kind != PK_GEMM) {
        lazy_pdl();
        if (warp == kEpilogueWarp0 && P.n_deps) {
#ifdef IOS_ROW_BANDS
          int g0, g1;
          simt_rows(P, views[P.in_begin].H, t - P.tile_begin, g0, g1);
          wait_deps(P, bands, counters, err, ep, lane, g0, g1);
#else
          wait_deps(P, counters, err, ep, lane);
#endif
        }
        named_bar(2, 128);
#ifndef IOS_NO_SIMT
        simt_tile<DT>(P, views, t - P.tile_begin, etid, 128);
#endif
        named_bar(2, 128);
        if (etid == 0 && P.signal) {
          red_release_add(counters + P.done_idx, 1);
          IOS_BAND_SIGNAL(t - P.tile_begin);
        }
        continue;
      }
      const int local = t - P.tile_begin;
      const int rest = fdiv(P.fd_split, local);
      const int s = local - rest * P.split;
      const int mt = fdiv(P.fd_ntn, rest);
      const int nt = rest - mt * P.n_tiles_n;
      // tile row -> output pixel (-1: none). Dense tiles: 128 consecutive pixels. Tap-TMA tiles:
      // a tN x tR x tWt output patch, row r = (nn * tR + i) * tWt + j.
      int tn0 = 0, toh0 = 0, tow0 = 0;
      if (P.tt) {
        const int rr = fdiv(P.fd_tilw, mt);
        const int tw = mt - rr * P.tiles_w;
        const int tnn = fdiv(P.fd_tilh, rr);
        tn0 = tnn * P.tN;
        toh0 = (rr - tnn * P.tiles_h) * P.tR;
        tow0 = tw * P.tWt;
      }
      const int trows = P.tt ? P.tN * P.tR * P.tWt : min(kBM, P.M - mt * kBM);
      // everything the store loops need is copied into registers: the descriptors are read through
      // generic pointers, and a descriptor re-load behind a global store waits for that store
      const bool is_tt = P.tt != 0;
      const FastDiv fthw = P.fd_thw, ftw = P.fd_tw;
      const int thw = P.tR * P.tWt, tWt = P.tWt, nb = P.batch, Ho = P.Ho, Wo = P.Wo, Mx = P.M, BNx = P.BN;
      auto pixel = [=](int r) -> int {
        if (!is_tt) return r < trows ? mt * kBM + r : -1;
        const int nn = fdiv(fthw, r);
        const int rem = r - nn * thw;
        const int i = fdiv(ftw, rem);
        const int n = tn0 + nn, oh = toh0 + i, ow = tow0 + rem - i * tWt;
        return (r < trows && n < nb && oh < Ho && ow < Wo) ? (n * Ho + oh) * Wo + ow : -1;
      };
      const float* bias = reinterpret_cast<const float*>(P.bias);
      if (P.swap_ab) {
        // swap-AB tile: TMEM lane = output channel, columns = pixels. Each thread owns one channel;
        // a warp's stores/reductions for one pixel cover 32 consecutive channels (coalesced).
        const int ch = mt * kBM + etid;   // column of the (merged) GEMM
        const Segment* sgp = nullptr;
        for (int q = 0; q < P.n_seg; ++q) {
          const Segment& sg = segs[P.seg_begin + q];
          if (ch >= sg.n0 && ch < sg.n1) sgp = &sg;
        }
        const float bv = sgp ? __ldg(bias + ch) : 0.f;
        const int relu = sgp ? sgp->relu : 0;
        // Output writes go through this warp's smem staging area as 16 B vectors along channels:
        // per 4 pixels each thread stages its channel's 4 values ([pixel][32 channels]), then lane
        // (pixel p, 16 B piece q) stores one vector. Lane q's destination comes from the segment of
        // its own piece (segment boundaries are multiples of 8 channels).
        constexpr int OESZ = DT == ET_BF16 ? 2 : 4;
        constexpr int PPP = 32 * OESZ / 16;           // 16 B pieces per pixel row of 32 channels (8 / 4)
        const uint32_t stg = smem_u32(sepi) + (warp & 3) * 4096;
        const int sp = lane / PPP, sq = lane % PPP;   // store lane -> (pixel in the group, piece)
        char* qptr = nullptr;
        int64_t qstride = 0;
        {
          const int qch = mt * kBM + (warp & 3) * 32 + sq * (16 / OESZ);
          for (int q = 0; q < P.n_seg; ++q) {
            const Segment& sg = segs[P.seg_begin + q];
            if (qch >= sg.n0 && qch < sg.n1) {
              qptr = reinterpret_cast<char*>(sg.out.ptr) + ((int64_t)sg.out.coff + qch - sg.n0) * OESZ;
              qstride = (int64_t)sg.out.cstride * OESZ;
            }
          }
        }
        // stage 4 pixels (px0 .. px0+3) of this thread's channel, then store them as vectors
        auto emit4 = [&](int px0, const float* o) {
          if (DT == ET_BF16) {
#pragma unroll
            for (int e = 0; e < 4; ++e)
              asm volatile("st.shared.b16 [%0], %1;" ::"r"(stg + (e * 32 + lane) * 2), "h"(bf16_bits(o[e])));
          } else {
#pragma unroll
            for (int e = 0; e < 4; ++e)
              asm volatile("st.shared.b32 [%0], %1;" ::"r"(stg + (e * 32 + lane) * 4), "r"(__float_as_uint(rnd(o[e], DT))));
          }
          __syncwarp();
          if (sp < 4 && qptr && px0 + sp < Mx) {
            uint32_t w0, w1, w2, w3;
            asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(w0), "=r"(w1), "=r"(w2), "=r"(w3)
                         : "r"(stg + sp * 32 * OESZ + sq * 16));
            stg_v4(qptr + (int64_t)(px0 + sp) * qstride, w0, w1, w2, w3);
          }
          __syncwarp();
        };
        mbar_wait(smem_u32(&tfull[acc]), acc_phase);
        lazy_pdl();
        if (etid == 0 && tfirst) IOS_TRACE(5);
        tc_fence_after();
        const uint32_t tbase = tmem_base + ((uint32_t)lane_base << 16) + (uint32_t)acc * kMaxBN;
        const int out_tile = mt;
        if (P.split == 1) {
          // 16 pixels per round: this thread's channel of each staged as [pixel][32 channels], one
          // warp sync, then every lane stores pixels (lane / PPP) + k * (32 / PPP) of its piece
          for (int c0 = 0; c0 < BNx && c0 < Mx; c0 += 16) {
            uint32_t v[16];
            tmem_ld16(tbase + c0, v);
            tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 16; ++e) {
              float o = __uint_as_float(v[e]) + bv;
              if (relu) o = fmaxf(o, 0.f);
              if (DT == ET_BF16)
                asm volatile("st.shared.b16 [%0], %1;" ::"r"(stg + (e * 32 + lane) * 2), "h"(bf16_bits(o)));
              else
                asm volatile("st.shared.b32 [%0], %1;" ::"r"(stg + (e * 32 + lane) * 4), "r"(__float_as_uint(rnd(o, DT))));
            }
            __syncwarp();
#pragma unroll
            for (int k = 0; k < 16 / (32 / PPP); ++k) {
              const int px = sp + k * (32 / PPP);
              if (qptr && c0 + px < Mx) {
                uint32_t w0, w1, w2, w3;
                asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(w0), "=r"(w1), "=r"(w2), "=r"(w3)
                             : "r"(stg + px * 32 * OESZ + sq * 16));
                stg_v4(qptr + (int64_t)(c0 + px) * qstride, w0, w1, w2, w3);
              }
            }
            __syncwarp();
          }
          tc_fence_before();
          mbar_arrive(smem_u32(&tempty[acc]));
        } else {
          // split-K: fp32 accumulator channel-major [128 channels][BN pixels]; each thread adds its
          // channel's 16 pixels per TMEM load with four 16 B vector reductions (pixels past M add 0)
          // split s writes its partial into its own slab [S][128][BN] of the tile (plain stores:
          // L2 write bandwidth, no atomics); the finalize sums the S slabs in a fixed order
          // (deterministic)
          const int64_t slab = (int64_t)kBM * BNx;
          const bool slabs = P.slabs != 0;   // else: vector reductions into one zeroed slab
          float* tacc = reinterpret_cast<float*>(P.workspace) + (int64_t)out_tile * slab * (slabs ? P.split : 1);
          float* trow = tacc + (int64_t)etid * BNx;
          float* mrow = trow + (slabs ? s * slab : 0);
          // the splits of a tile reduce into the same lines: each starts at a different 16-column
          // round (rotation by split index) so they do not queue on the same L2 lines at once
          const int nr16 = (BNx + 15) >> 4;
          for (int k = 0; k < nr16; ++k) {
            const int c0 = ((k + s) % nr16) * 16;
            uint32_t v[16];
            tmem_ld16(tbase + c0, v);
            tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 16; ++j)
              if (c0 + j >= Mx) v[j] = 0u;
#pragma unroll
            for (int q = 0; q < 4; ++q)
              if (c0 + 4 * q < Mx) {
                if (slabs)
                  stg_v4(mrow + c0 + 4 * q, v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
                else
                  red_add_v4(mrow + c0 + 4 * q, v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
              }
          }
          tc_fence_before();
          mbar_arrive(smem_u32(&tempty[acc]));
          named_bar(2, 128);
          if (warp == kEpilogueWarp0) split_rendezvous(counters + P.tilectr_idx + out_tile, P.split, err, ep, lane);
          named_bar(2, 128);
          // distributed finalize: split s owns pixel quads [s*np4/S, (s+1)*np4/S) of the tile; each
          // thread sums its channel's quads over the S slabs (16 float4 in flight) and emits them
          // through the staged vector stores. Reading lines other SMs just reduced into is slow,
          // so the S splits share the read-back instead of one last-arriving CTA doing it all.
          const int np4 = (Mx + 3) >> 2;
          const int kq0 = s * np4 / P.split, kq1 = (s + 1) * np4 / P.split;
          if (etid == 0) IOS_TRACE(13);
          for (int k0 = kq0; k0 < kq1; k0 += 4) {
            float4 x[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) x[u] = make_float4(0.f, 0.f, 0.f, 0.f);
            const int nsl = slabs ? P.split : 1;
            for (int j0 = 0; j0 < nsl; j0 += 4) {   // 4 quads x 4 slabs in flight
              float4 t[4][4];
#pragma unroll
              for (int jj = 0; jj < 4; ++jj)
#pragma unroll
                for (int u = 0; u < 4; ++u)
                  t[jj][u] = (j0 + jj < nsl && k0 + u < kq1)
                                 ? __ldcg(reinterpret_cast<const float4*>(trow + (j0 + jj) * slab) + k0 + u)
                                 : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
              for (int jj = 0; jj < 4; ++jj)
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                  x[u].x += t[jj][u].x; x[u].y += t[jj][u].y; x[u].z += t[jj][u].z; x[u].w += t[jj][u].w;
                }
            }
            if (etid == 0 && k0 == kq0) IOS_TRACE(14);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              if (k0 + u >= kq1) break;
              if (!slabs) stg_zero4_cg(reinterpret_cast<float4*>(trow) + k0 + u);   // re-zero for the next launch
              float o[4] = {x[u].x + bv, x[u].y + bv, x[u].z + bv, x[u].w + bv};
              if (relu) {
#pragma unroll
                for (int e = 0; e < 4; ++e) o[e] = fmaxf(o[e], 0.f);
              }
              emit4((k0 + u) * 4, o);
            }
          }
          if (etid == 0) IOS_TRACE(15);
        }
        if (P.signal) {
          named_bar(2, 128);
          if (etid == 0) {
            red_release_add(counters + P.done_idx, 1);
            IOS_BAND_SIGNAL(mt);
          }
        }
        tfirst = false;
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1u;
        continue;
      }
      // FP32-SIMT mode: the epilogue warps are the GEMM consumer: thread = tile row, BN <= 32
      // columns in registers, exact fp32 FMA over every K chunk the producers stage
      float sacc[32];
#pragma unroll
      for (int e = 0; e < 32; ++e) sacc[e] = 0.f;
      if constexpr (DT == ET_F32X) {
        const int c0 = s * P.chunks_per_split;
        const int c1 = min(c0 + P.chunks_per_split, P.k_chunks);
        const int bn = BNx;
        for (int c = c0; c < c1; ++c) {
          mbar_wait(smem_u32(&full[ering.slot]), ering.phase);
          const uint8_t* As = slotA(ering.slot) + (etid >> 3) * 1024 + (etid & 7) * 16;
          const uint8_t* Bs = slotB(ering.slot);
          float a[32];
#pragma unroll
          for (int pc = 0; pc < 8; ++pc) {
            const float4 v = *reinterpret_cast<const float4*>(As + pc * 128);
            a[4 * pc] = v.x; a[4 * pc + 1] = v.y; a[4 * pc + 2] = v.z; a[4 * pc + 3] = v.w;
          }
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            if (j >= bn) break;
            const uint8_t* brow = Bs + (j >> 3) * 1024 + (j & 7) * 16;
            float accj = sacc[j];
#pragma unroll
            for (int pc = 0; pc < 8; ++pc) {
              const float4 b = *reinterpret_cast<const float4*>(brow + pc * 128);   // broadcast
              accj = fmaf(a[4 * pc], b.x, accj);
              accj = fmaf(a[4 * pc + 1], b.y, accj);
              accj = fmaf(a[4 * pc + 2], b.z, accj);
              accj = fmaf(a[4 * pc + 3], b.w, accj);
            }
            sacc[j] = accj;
          }
          named_bar(2, 128);
          if (etid == 0) mbar_arrive(smem_u32(&empty[ering.slot]));   // slot free for the producers
          ering.next();
        }
      }
      // stage this tile's bias slice in smem while the MMAs run (one load round trip, off the
      // critical path); the previous tile's readers of this buffer are past the barrier below
      float* sbias = sbias_all + acc * kMaxBN;
      for (int i = etid; i < BNx; i += 128) sbias[i] = __ldg(bias + nt * BNx + i);
      named_bar(2, 128);
      if (DT != ET_F32X) mbar_wait(smem_u32(&tfull[acc]), acc_phase);
      lazy_pdl();
      if (etid == 0 && tfirst) IOS_TRACE(5);
      tc_fence_after();
      const uint32_t tbase = tmem_base + ((uint32_t)lane_base << 16) + (uint32_t)acc * kMaxBN;
      const int out_tile = mt * P.n_tiles_n + nt;
      // ---- cluster split-K: the csplit CTAs of this tile's group (consecutive cluster ranks) sum
      // their partials in shared memory. Rank r owns rows [r * 128 / cD, (r + 1) * 128 / cD): those
      // are the TMEM lanes of its epilogue warps q with q * cD / 4 == r. Every other warp pushes its
      // 32 rows x BN fp32 into the owner's receive buffer (slot j = the sender's rank among the
      // others), st.async completing bytes on the owner's rfull; the owner adds the cD - 1 received
      // rows to its own before the store (or, with more splits than cD, before the global reduction).
      int cD = 1;
      bool c_owner = true;
      uint32_t c_rbuf = 0;                   // this owner thread's row in receive slot 0
      uint32_t c_rank = 0, c_gbase = 0;      // own cluster rank; cluster rank of the group's rank 0
      int c_slot = 0;                        // bytes between receive slots
      if constexpr (kCsk) {
        if (P.csplit > 1) {
          cD = P.csplit;
          const int r = s % cD;
          c_rank = cluster_rank();
          c_gbase = c_rank - (uint32_t)r;
          const int q = warp & 3, o = q * cD / 4;
          const int rows_per = kBM / cD;
          const int rr = (q - o * 4 / cD) * 32 + lane;     // row inside the owner's band
          const uint32_t rbuf0 = smem_u32(smem + sd.rbuf_off);
          c_slot = rows_per * sd.rbuf_stride;
          c_owner = o == r;
          if (!c_owner) {
            const uint32_t oc = c_gbase + (uint32_t)o;
            mbar_wait_cluster(smem_u32(&sempty[oc]), ((csk_sbits >> oc) & 1u) ^ 1u);
            const int j = r < o ? r : r - 1;
            const uint32_t rrow = mapa(rbuf0 + (uint32_t)(j * c_slot + rr * sd.rbuf_stride), oc);
            const uint32_t rbar = mapa(smem_u32(rfull), oc);
            for (int c0 = 0; c0 < BNx; c0 += 16) {
              uint32_t v[16];
              tmem_ld16(tbase + c0, v);
              tmem_ld_wait();
#pragma unroll
              for (int i = 0; i < 4; ++i)
                st_async_v4(rrow + (uint32_t)(c0 + 4 * i) * 4u, rbar, v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
            }
          } else {
            c_rbuf = rbuf0 + (uint32_t)(rr * sd.rbuf_stride);
            if (lane == 0 && q == r * 4 / cD)
              mbar_arrive_expect_tx(smem_u32(rfull), (uint32_t)((cD - 1) * rows_per * BNx * 4));
          }
          for (int k = 0; k < cD; ++k)
            if (k != r) csk_sbits ^= 1u << (c_gbase + (uint32_t)k);
          if (c_owner) mbar_wait_cluster(smem_u32(rfull), csk_rphase);
          csk_rphase ^= 1u;
        }
      }
      // owner: add the cD - 1 received partials of this thread's row, columns [c0, c0 + 32)
      auto add_received = [&](int c0, float* o) {
        if constexpr (kCsk) {
          for (int j = 0; j < cD - 1; ++j) {
            const uint32_t a = c_rbuf + (uint32_t)(j * c_slot + c0 * 4);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              uint32_t w0, w1, w2, w3;
              asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(w0), "=r"(w1), "=r"(w2), "=r"(w3) : "r"(a + 16 * i));
              o[4 * i] += __uint_as_float(w0);
              o[4 * i + 1] += __uint_as_float(w1);
              o[4 * i + 2] += __uint_as_float(w2);
              o[4 * i + 3] += __uint_as_float(w3);
            }
          }
        }
      };
      if (P.split == cD) {
        // Per 32-column round: TMEM -> registers (thread = row) -> bias/rounding -> this warp's 4 KB
        // smem staging tile (16 B pieces XOR-swizzled by row: conflict-free) -> coalesced 16 B global
        // stores (lanes sweep a row's contiguous channels; 4 rows per instruction) instead of 32
        // scattered rows. A merged conv's columns belong to several output segments (branches,
        // P:193 split): segments are multiples of 8 channels, so every 16 B piece lies in one segment;
        // each lane looks up its piece's segment once per round and applies that branch's ReLU
        // (after rounding: max(0, rnd(x)) == rnd(max(0, x)) for TF32 and bf16).
        constexpr int OESZ = DT == ET_BF16 ? 2 : 4;
        constexpr int PPR = 32 * OESZ / 16;                 // 16 B pieces per row per round (8 / 4)
        const uint32_t stg = smem_u32(sepi) + (warp & 3) * 4096;
        constexpr int RPI = 32 / PPR;                       // rows per write-out instruction (4 / 8)
        int opix[32 / RPI];                                 // output pixel of each row this lane writes
        if (!is_tt) {
#pragma unroll
          for (int it = 0; it < 32 / RPI; ++it) opix[it] = pixel((warp & 3) * 32 + it * RPI + lane / PPR);
        } else {
          // patch tile: decode the lane's first row once, then step RPI rows (j, i, nn carry) instead
          // of two divisions per row
          const int r0 = (warp & 3) * 32 + lane / PPR;
          int nn = fdiv(fthw, r0);
          int rem = r0 - nn * thw;
          int i = fdiv(ftw, rem), j = rem - i * tWt;
          const int tRr = P.tR;
#pragma unroll
          for (int it = 0; it < 32 / RPI; ++it) {
            const int r = r0 + it * RPI, n = tn0 + nn, oh = toh0 + i, ow = tow0 + j;
            opix[it] = (r < trows && n < nb && oh < Ho && ow < Wo) ? (n * Ho + oh) * Wo + ow : -1;
            j += RPI;
            while (j >= tWt) {
              j -= tWt;
              if (++i == tRr) {
                i = 0;
                ++nn;
              }
            }
          }
        }
        const int sg0 = P.seg_begin, nsg = P.n_seg;
        // one output segment (every conv but a merged one): its destination once per tile
        char* s1_base = nullptr;
        int s1_n0 = 0, s1_n1 = 0, s1_cs = 0, s1_relu = 0;
        if (nsg == 1) {
          const Segment& sg = segs[sg0];
          s1_n0 = sg.n0;
          s1_n1 = sg.n1;
          s1_cs = sg.out.cstride;
          s1_relu = sg.relu;
          s1_base = reinterpret_cast<char*>(sg.out.ptr) + ((int64_t)sg.out.coff - sg.n0) * OESZ;
        }
        for (int c0 = 0; c_owner && c0 < BNx; c0 += 32) {
          uint32_t va[16], vb[16];
          acc_ld16<DT>(tbase + c0, sacc, c0, va);
          acc_ld16<DT>(tbase + c0 + 16, sacc, c0 + 16, vb);
          acc_wait<DT>();
#ifndef IOS_TRACE_FINE
          if (etid == 0 && tfirst && c0 == 0) IOS_TRACE(13);
#endif
          float o[32];
#pragma unroll
          for (int e = 0; e < 32; ++e) o[e] = __uint_as_float(e < 16 ? va[e] : vb[e - 16]);
          if (kCsk && cD > 1) add_received(c0, o);
          {
            const float4* sb4 = reinterpret_cast<const float4*>(sbias + c0);   // 16 B aligned
#pragma unroll
            for (int e4 = 0; e4 < 8; ++e4) {
              const float4 b4 = sb4[e4];
              o[4 * e4] += b4.x;
              o[4 * e4 + 1] += b4.y;
              o[4 * e4 + 2] += b4.z;
              o[4 * e4 + 3] += b4.w;
            }
          }
#pragma unroll
          for (int p = 0; p < PPR; ++p) {
            uint32_t w[4];
            if (DT == ET_BF16) {
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                __nv_bfloat162 h = __floats2bfloat162_rn(o[p * 8 + 2 * q], o[p * 8 + 2 * q + 1]);
                w[q] = *reinterpret_cast<uint32_t*>(&h);
              }
            } else {
#pragma unroll
              for (int q = 0; q < 4; ++q) w[q] = __float_as_uint(rnd(o[p * 4 + q], DT));
            }
            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(stg + lane * (PPR * 16) + ((p ^ (lane & 7)) % PPR) * 16),
                         "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]) : "memory");
          }
          __syncwarp();
#ifndef IOS_TRACE_FINE
          if (etid == 0 && tfirst && c0 == 0) IOS_TRACE(14);
#endif
          // this lane's piece column and its segment (destination, channel stride, ReLU)
          const int p = lane % PPR;
          const int ncol = nt * BNx + c0 + p * (16 / OESZ);
          char* dst = nullptr;
          int ocs = 0, relu = 0;
          // (columns past BN in the last round belong to the next N tile: never written from here)
          if (nsg == 1) {
            if (c0 + p * (16 / OESZ) < BNx && ncol >= s1_n0 && ncol < s1_n1) {
              dst = s1_base + (int64_t)ncol * OESZ;
              ocs = s1_cs;
              relu = s1_relu;
            }
          } else {
            for (int q = 0; q < nsg && c0 + p * (16 / OESZ) < BNx; ++q) {
              const Segment& sg = segs[sg0 + q];
              if (ncol >= sg.n0 && ncol < sg.n1) {
                dst = reinterpret_cast<char*>(sg.out.ptr) + ((int64_t)sg.out.coff + ncol - sg.n0) * OESZ;
                ocs = sg.out.cstride;
                relu = sg.relu;
              }
            }
          }
          // coalesced write-out: lane -> (row, piece)
#pragma unroll
          for (int it = 0; it < 32 / RPI; ++it) {
            const int r = it * RPI + lane / PPR;
            uint32_t w[4];
            asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3])
                         : "r"(stg + r * (PPR * 16) + ((p ^ (r & 7)) % PPR) * 16));
            if (relu) {
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                if (DT == ET_BF16) {
                  __nv_bfloat162 h = *reinterpret_cast<__nv_bfloat162*>(&w[q]);
                  h = __hmax2(h, __floats2bfloat162_rn(0.f, 0.f));
                  w[q] = *reinterpret_cast<uint32_t*>(&h);
                } else {
                  w[q] = __float_as_uint(fmaxf(__uint_as_float(w[q]), 0.f));
                }
              }
            }
            if (opix[it] >= 0 && dst) stg_v4(dst + (int64_t)opix[it] * ocs * OESZ, w[0], w[1], w[2], w[3]);
          }
          __syncwarp();
#ifndef IOS_TRACE_FINE
          if (etid == 0 && tfirst && c0 == 0) IOS_TRACE(15);
#endif
        }
        tc_fence_before();
        if (DT != ET_F32X) mbar_arrive(smem_u32(&tempty[acc]));
      } else {
        // split-K: every split stores its fp32 partial into its own slab of the tile (plain
        // coalesced stores; L2 atomics were throughput-bound), all splits rendezvous, and each
        // finalizes 1/S of the tile: sum of the S slabs in split order (deterministic), bias/ReLU.
        float* ws = reinterpret_cast<float*>(P.workspace);
        const int64_t slab = (int64_t)kBM * BNx;
        const bool slabs = P.slabs != 0;                         // else: reductions into one zeroed slab
        float* tacc = ws + (int64_t)out_tile * slab * (slabs ? P.split : 1);  // [S][kBM][BN] fp32 partials
        float* macc = tacc + (slabs ? s * slab : 0);            // this split's slab
        const uint32_t stg = smem_u32(sepi) + (warp & 3) * 4096;
        const int wr0 = (warp & 3) * 32;
        // the splits of a tile reduce into the same lines: rotate the 32-column round and the 4-row
        // group order by split index so they do not queue on the same L2 lines at the same time
        const int nr32 = (BNx + 31) >> 5;
        const int ks = nr32 == 1 ? 0 : (int)((uint32_t)s % (uint32_t)nr32);   // (once per tile, not per round)
        for (int k = 0; c_owner && k < nr32; ++k) {
          const int c0 = (k + ks < nr32 ? k + ks : k + ks - nr32) * 32, rot = s;
          uint32_t va[16], vb[16];
          acc_ld16<DT>(tbase + c0, sacc, c0, va);
          acc_ld16<DT>(tbase + c0 + 16, sacc, c0 + 16, vb);
          acc_wait<DT>();
          if (kCsk && cD > 1) {   // this owner's rows: the group's csplit partials summed first
            float o[32];
#pragma unroll
            for (int e = 0; e < 32; ++e) o[e] = __uint_as_float(e < 16 ? va[e] : vb[e - 16]);
            add_received(c0, o);
#pragma unroll
            for (int e = 0; e < 16; ++e) {
              va[e] = __float_as_uint(o[e]);
              vb[e] = __float_as_uint(o[16 + e]);
            }
          }
          // stage (swizzled) then coalesced vector reductions: 4 rows x 128 B per instruction
#pragma unroll
          for (int p = 0; p < 8; ++p) {
            const uint32_t* src = p < 4 ? va + p * 4 : vb + (p - 4) * 4;
            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(stg + lane * 128 + ((p ^ (lane & 7)) * 16)),
                         "r"(src[0]), "r"(src[1]), "r"(src[2]), "r"(src[3]) : "memory");
          }
          __syncwarp();
#pragma unroll
          for (int it = 0; it < 8; ++it) {
            const int r = ((it + rot) & 7) * 4 + lane / 8, p = lane % 8;
            uint32_t w0, w1, w2, w3;
            asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(w0), "=r"(w1), "=r"(w2), "=r"(w3)
                         : "r"(stg + r * 128 + ((p ^ (r & 7)) * 16)));
            const int col = c0 + p * 4;
            if (wr0 + r < trows && col < BNx) {
              if (slabs)
                stg_v4(macc + (wr0 + r) * BNx + col, w0, w1, w2, w3);
              else
                red_add_v4(macc + (wr0 + r) * BNx + col, w0, w1, w2, w3);
            }
          }
          __syncwarp();
        }
        tc_fence_before();
        if (DT != ET_F32X) mbar_arrive(smem_u32(&tempty[acc]));
        named_bar(2, 128);
#ifndef IOS_TRACE_FINE
        if (etid == 0 && tfirst) IOS_TRACE(13);
#endif
        if (warp == kEpilogueWarp0) split_rendezvous(counters + P.tilectr_idx + out_tile, P.split, err, ep, lane);
        named_bar(2, 128);
#ifndef IOS_TRACE_FINE
        if (etid == 0 && tfirst) IOS_TRACE(14);
#endif
        {
          // distributed finalize (see the swap-AB path): split s owns tile rows
          // [s*trows/S, (s+1)*trows/S); all 128 threads, coalesced (consecutive threads sweep a
          // row's contiguous columns)
          const int bn = BNx, q4 = bn / 4;
          const FastDiv fq4 = P.fd_q4;
          const int r0 = fdiv(P.fd_split, s * trows), r1 = fdiv(P.fd_split, (s + 1) * trows);   // s*trows/S
          const int total = (r1 - r0) * q4;
          // one output segment (every conv but a merged one): destination fields once per tile
          const bool seg1 = P.n_seg == 1;
          const Segment& sg1 = segs[P.seg_begin];
          const int f1_n0 = sg1.n0, f1_n1 = sg1.n1, f1_cs = sg1.out.cstride, f1_relu = sg1.relu;
          char* const f1_base = reinterpret_cast<char*>(sg1.out.ptr) + ((int64_t)sg1.out.coff - sg1.n0) * (DT == ET_BF16 ? 2 : 4);
          // 4 elements x 4 slabs = 16 independent float4 loads in flight per thread
          for (int base = etid; base < total; base += 128 * 4) {
            float4 x[4];
            int off[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int idx = base + u * 128;
              const int qr = fdiv(fq4, idx);   // (idx / q4 by multiply-shift: q4 = BN / 4)
              off[u] = idx < total ? (r0 + qr) * bn + (idx - qr * q4) * 4 : -1;
              x[u] = make_float4(0.f, 0.f, 0.f, 0.f);
            }
            const int nsl = slabs ? P.split : 0;
            if (!slabs) {   // one reduced slab: 4 independent loads
#pragma unroll
              for (int u = 0; u < 4; ++u)
                if (off[u] >= 0) x[u] = __ldcg(reinterpret_cast<const float4*>(tacc + off[u]));
            }
            for (int j0 = 0; j0 < nsl; j0 += 4) {
              float4 t[4][4];
#pragma unroll
              for (int jj = 0; jj < 4; ++jj)
#pragma unroll
                for (int u = 0; u < 4; ++u)
                  t[jj][u] = (j0 + jj < nsl && off[u] >= 0)
                                 ? __ldcg(reinterpret_cast<const float4*>(tacc + (j0 + jj) * slab + off[u]))
                                 : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
              for (int jj = 0; jj < 4; ++jj)
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                  x[u].x += t[jj][u].x; x[u].y += t[jj][u].y; x[u].z += t[jj][u].z; x[u].w += t[jj][u].w;
                }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int idx = base + u * 128;
              if (idx >= total) break;
              const int qr = fdiv(fq4, idx);
              const int r = r0 + qr, col = (idx - qr * q4) * 4;
              if (!slabs) stg_zero4_cg(tacc + off[u]);   // re-zero for the next launch
              const int ncol = nt * bn + col;
              int n0 = f1_n0, n1 = f1_n1, ocs = f1_cs, relu = f1_relu;
              char* obase = f1_base;
              if (!seg1) {
                for (int q = 0; q < P.n_seg; ++q) {
                  const Segment& sg = segs[P.seg_begin + q];
                  if (ncol >= sg.n0 && ncol < sg.n1) {
                    n0 = sg.n0;
                    n1 = sg.n1;
                    ocs = sg.out.cstride;
                    relu = sg.relu;
                    obase = reinterpret_cast<char*>(sg.out.ptr) + ((int64_t)sg.out.coff - sg.n0) * (DT == ET_BF16 ? 2 : 4);
                    break;
                  }
                }
              }
              if (ncol < n0 || ncol >= n1) continue;
              const int px = pixel(r);
              if (px < 0) continue;
              float o[4] = {x[u].x + sbias[col], x[u].y + sbias[col + 1], x[u].z + sbias[col + 2], x[u].w + sbias[col + 3]};
              if (relu) {
#pragma unroll
                for (int e = 0; e < 4; ++e) o[e] = fmaxf(o[e], 0.f);
              }
              const int64_t eoff = (int64_t)px * ocs + ncol;   // elements from obase
              if (DT == ET_BF16) {
                __nv_bfloat162 h0 = __floats2bfloat162_rn(o[0], o[1]), h1 = __floats2bfloat162_rn(o[2], o[3]);
                stg_v2(reinterpret_cast<__nv_bfloat16*>(obase) + eoff, *reinterpret_cast<uint32_t*>(&h0),
                       *reinterpret_cast<uint32_t*>(&h1));
              } else {
                stg_v4(reinterpret_cast<float*>(obase) + eoff, __float_as_uint(rnd(o[0], DT)), __float_as_uint(rnd(o[1], DT)),
                       __float_as_uint(rnd(o[2], DT)), __float_as_uint(rnd(o[3], DT)));
              }
            }
          }
        }
      }
      if (P.signal || cD > 1) {
        named_bar(2, 128);
        if (etid == 0) {
          if constexpr (kCsk) {
            // this CTA's receive buffer is consumed: release it to every other rank of the group
            const uint32_t mine = smem_u32(&sempty[c_rank]);
            for (int k = 0; k < cD; ++k)
              if (c_gbase + (uint32_t)k != c_rank) mbar_arrive_remote(mapa(mine, c_gbase + (uint32_t)k));
          }
          if (P.signal) {
            red_release_add(counters + P.done_idx, 1);
            IOS_BAND_SIGNAL(mt);
          }
        }
      }
      tfirst = false;
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1u;
    }
  }

  if (kTrace && trace && (tid == kEpilogueWarp0 * 32 || tid == kMmaWarp * 32))
    IOS_TRACE(tid == kMmaWarp * 32 ? 4 : 6);
  // ---------------------------------------------------------------------------- teardown
  __syncwarp();   // the MMA warp ran its loop on lane 0 only
  tc_fence_before();
  // a cluster launch: no CTA leaves while a peer may still arrive on its barriers
  if (csk_launch)
    cluster_sync_all();
  else
    __syncthreads();
  if (warp == kMmaWarp && sd.has_gemm && DT != ET_F32X) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(kTmemCols) : "memory");
  }
  if (tid == 0) {
    IOS_TRACE(7);   // counters are epoch-relative: nothing to reset at exit
    IOS_TRACE(8);
    if (sd.stamp) atomicMax(reinterpret_cast<unsigned long long*>(sd.stamp) + 1, (unsigned long long)gtimer());
  }
#undef IOS_TRACE
}

#ifdef IOS_INST_DT
#define IOS_LAUNCHER_DEF3(dt, sdv, ft) IOS_LAUNCHER_DECL(dt, sdv, ft)
#define IOS_LAUNCHER_DECL(dt, sdv, ft) \
  cudaError_t launch_stage_inst_##dt##_##sdv##_##ft(cudaLaunchConfig_t& cfg, const StageDesc& sd)
IOS_LAUNCHER_DEF3(IOS_INST_DT, IOS_INST_SD, IOS_INST_FEAT) {
  static bool attr_done = false;
  static int max_grid = 0, max_cluster_grid = 0;
  auto k = ios_stage_kernel<IOS_INST_DT, (IOS_INST_SD != 0), IOS_INST_FEAT>;
  if (!attr_done) {
    cudaError_t e = cudaFuncSetAttribute((const void*)k, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes + 1024);
    if (e != cudaSuccess) return e;
    // co-residency: the in-kernel dependency waits assume every CTA of the grid is resident at
    // once (one per SM); refuse a grid the device cannot hold instead of spinning into the guard
    int per_sm = 0, dev = 0, sms = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void*)k, kThreads, kSmemBytes + 1024);
    if (e != cudaSuccess) return e;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    max_grid = per_sm * sms;
    if ((IOS_INST_FEAT & F_CSK) != 0) {
      // clusters of kClusterCtas one-CTA-per-SM blocks fit fewer SMs than the plain grid (GPC sizes)
      cudaLaunchConfig_t q = cfg;
      cudaLaunchAttribute a[1];
      a[0].id = cudaLaunchAttributeClusterDimension;
      a[0].val.clusterDim.x = kClusterCtas;
      a[0].val.clusterDim.y = 1;
      a[0].val.clusterDim.z = 1;
      q.attrs = a;
      q.numAttrs = 1;
      q.gridDim = dim3(kClusterCtas * 8);
      int nc = 0;
      e = cudaOccupancyMaxActiveClusters(&nc, (const void*)k, &q);
      if (e != cudaSuccess) return e;
      max_cluster_grid = nc * kClusterCtas;
    }
    attr_done = true;
  }
  bool cluster = false;
  for (unsigned i = 0; i < cfg.numAttrs; ++i) cluster |= cfg.attrs[i].id == cudaLaunchAttributeClusterDimension;
  if ((int)(cfg.gridDim.x) > (cluster ? max_cluster_grid : max_grid)) return cudaErrorCooperativeLaunchTooLarge;
  return cudaLaunchKernelEx(&cfg, k, sd);
}
#if IOS_INST_DT == 0 && IOS_INST_SD == 1 && IOS_INST_FEAT == 8   // (F_CSK: an enum, not visible to #if)
// co-resident CTAs of a cluster launch (clusters of kClusterCtas, one CTA per SM); 0 on error
int stage_cluster_ctas() {
  auto k = ios_stage_kernel<0, true, F_CSK>;
  if (cudaFuncSetAttribute((const void*)k, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes + 1024) != cudaSuccess)
    return 0;
  cudaLaunchConfig_t q{};
  q.gridDim = dim3(kClusterCtas * 8);
  q.blockDim = dim3(kThreads);
  q.dynamicSmemBytes = kSmemBytes + 1024;
  cudaLaunchAttribute a[1];
  a[0].id = cudaLaunchAttributeClusterDimension;
  a[0].val.clusterDim.x = kClusterCtas;
  a[0].val.clusterDim.y = 1;
  a[0].val.clusterDim.z = 1;
  q.attrs = a;
  q.numAttrs = 1;
  int nc = 0;
  if (cudaOccupancyMaxActiveClusters(&nc, (const void*)k, &q) != cudaSuccess) return 0;
  return nc * kClusterCtas;
}
#endif

}  // namespace ios
#else
// ------------------------------------------------------------------------ boundary layout kernels
// 8 consecutive channels of one pixel as 16 B vector stores (32 B fp32 / 16 B bf16; C is padded to a
// multiple of 8, views are 16 B aligned: layout_ok)
__device__ __forceinline__ void store8(const View& vw, int dtype, int64_t pix, int c0, const float* v) {
  if (dtype != ET_BF16) {
    float* d = reinterpret_cast<float*>(vw.ptr) + pix * vw.cstride + vw.coff + c0;
    stg_v4(d, __float_as_uint(rnd(v[0], dtype)), __float_as_uint(rnd(v[1], dtype)), __float_as_uint(rnd(v[2], dtype)),
           __float_as_uint(rnd(v[3], dtype)));
    stg_v4(d + 4, __float_as_uint(rnd(v[4], dtype)), __float_as_uint(rnd(v[5], dtype)), __float_as_uint(rnd(v[6], dtype)),
           __float_as_uint(rnd(v[7], dtype)));
  } else {
    uint32_t w[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) w[q] = (uint32_t)bf16_bits(v[2 * q]) | ((uint32_t)bf16_bits(v[2 * q + 1]) << 16);
    stg_v4(reinterpret_cast<__nv_bfloat16*>(vw.ptr) + pix * vw.cstride + vw.coff + c0, w[0], w[1], w[2], w[3]);
  }
}

// NCHW fp32 (caller) -> NHWC padded (internal); rounds to the storage precision (Z14).
// Thread = (8-channel group g, pixel), pixel fastest: a warp reads 32 consecutive pixels of each of
// its 8 planes (coalesced) and writes 32 full 32 B sectors.
__global__ void nchw_to_nhwc_kernel(const float* __restrict__ in, View out, int dtype, int N, int C) {
  const int hw = out.H * out.W;
  const int npix = N * hw, ng = out.C / 8;
  const int total = npix * ng;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int g = i / npix, pix = i - g * npix;
    const int n = pix / hw, p = pix - n * hw;
    const float* src = in + (int64_t)n * C * hw + p;
    float v[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) v[e] = 8 * g + e < C ? __ldg(src + (int64_t)(8 * g + e) * hw) : 0.f;
    store8(out, dtype, pix, 8 * g, v);
  }
}

// NCHW fp32 (caller) -> the W-unfolded NHWC input of a narrow first conv (DeviceState::unfold):
// out pixel (n, h, ow), channel j * C + c = in[n, c, h, ow*sw - pw + j] (0 outside the image and in
// the padding channels), rounded to the storage precision. Thread = (8-channel group, output pixel).
__global__ void nchw_unfold_kernel(const float* __restrict__ in, View out, int dtype, int N, int C, int W, int kw, int sw,
                                   int pw) {
  const int ohw = out.H * out.W;
  const int npix = N * ohw, ng = out.C / 8;
  const int total = npix * ng;
  const int64_t hw = (int64_t)out.H * W;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int g = i / npix, pix = i - g * npix;
    const int n = pix / ohw, rem = pix - n * ohw;
    const int h = rem / out.W, ow = rem - h * out.W;
    const float* row = in + (int64_t)n * C * hw + (int64_t)h * W;
    const int w0 = ow * sw - pw;
    float v[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int ch = 8 * g + e;
      v[e] = 0.f;
      if (ch < kw * C) {
        const int j = ch / C, c = ch - j * C;
        const int w = w0 + j;
        if (w >= 0 && w < W) v[e] = __ldg(row + (int64_t)c * hw + w);
      }
    }
    store8(out, dtype, pix, 8 * g, v);
  }
}

// (32-bit indices: the launcher checks N * C * H * W < 2^31)
__global__ void nhwc_to_nchw_kernel(View in, int dtype, float* __restrict__ out, int N, int C) {
  const int hw = in.H * in.W;
  const int total = N * C * hw;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int nc = i / hw, p = i - nc * hw;
    const int n = nc / C, c = nc - n * C;
    out[i] = load_elem(in, dtype, (int64_t)n * hw + p, c);
  }
}

// Writes 2x the L2 size between profiler trials (Z15 l2_flush option).
__global__ void l2_flush_kernel(int4* buf, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    buf[i] = make_int4((int)i, 0, 0, 0);
}

// ------------------------------------------------------------------------------ host launchers
// The stage kernel's (dtype, smem-descriptor, feature class) instantiations are compiled as separate
// translation units (build.py passes -DIOS_INST_DT / _SD / _FEAT; nvcc runs them in parallel). Each
// unit exports one plain host launcher; launch_stage (host unit) dispatches to them.
#define IOS_LAUNCHER_DECL(dt, sdv, ft) \
  cudaError_t launch_stage_inst_##dt##_##sdv##_##ft(cudaLaunchConfig_t& cfg, const StageDesc& sd)
#define IOS_DECL_CLASSES(dt, sdv) \
  IOS_LAUNCHER_DECL(dt, sdv, 0); IOS_LAUNCHER_DECL(dt, sdv, 1); IOS_LAUNCHER_DECL(dt, sdv, 3); \
  IOS_LAUNCHER_DECL(dt, sdv, 8); IOS_LAUNCHER_DECL(dt, sdv, 9); IOS_LAUNCHER_DECL(dt, sdv, 11); IOS_LAUNCHER_DECL(dt, sdv, 15)
IOS_DECL_CLASSES(0, 0); IOS_DECL_CLASSES(0, 1); IOS_DECL_CLASSES(1, 0); IOS_DECL_CLASSES(1, 1);
IOS_LAUNCHER_DECL(2, 0, 3); IOS_LAUNCHER_DECL(2, 1, 3); IOS_LAUNCHER_DECL(2, 0, 15); IOS_LAUNCHER_DECL(2, 1, 15);

namespace {
// smallest compiled class covering the stage's features (FP32-SIMT: the full class only)
int feature_class(int dtype, int feat) {
  if (feat & F_TRACE) return kFeatTrace;
  int c = (dtype == ET_F32X || (feat & F_FDW)) ? kFeatFull : (feat & F_GATHER) ? kFeatGather : kFeatLean;
  if ((feat & F_CSK) && dtype != ET_F32X) c |= F_CSK;
  return c;
}
}  // namespace

cudaError_t launch_stage(const StageDesc& sd, int dtype, int grid, cudaStream_t st) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kSmemBytes + 1024;
  cfg.stream = st;
  cudaLaunchAttribute attr[3];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  // IOS_COOP=1: cooperative launch (the runtime guarantees co-residency of the whole grid or fails;
  // measured ~6 % slower end to end on Inception V3 b=1, so off by default)
  static const bool coop = getenv("IOS_COOP") && atoi(getenv("IOS_COOP")) != 0;
  if (coop) {
    attr[1].id = cudaLaunchAttributeCooperative;
    attr[1].val.cooperative = 1;
    cfg.numAttrs = 2;
  }
  // cluster split-K stages launch as clusters of kClusterCtas (grid a multiple of it)
  if (sd.cluster > 1) {
    attr[cfg.numAttrs].id = cudaLaunchAttributeClusterDimension;
    attr[cfg.numAttrs].val.clusterDim.x = (unsigned)sd.cluster;
    attr[cfg.numAttrs].val.clusterDim.y = 1;
    attr[cfg.numAttrs].val.clusterDim.z = 1;
    ++cfg.numAttrs;
  }
  const int sdv = sd.blob_bytes <= kDescBytes ? 1 : 0;
  const int fc = feature_class(dtype, sd.feat | (sd.trace ? F_TRACE : 0));
#define IOS_DISPATCH(dt, sv, f) \
  if (dtype == dt && sdv == sv && fc == f) return launch_stage_inst_##dt##_##sv##_##f(cfg, sd)
#define IOS_DISPATCH_ALL(dt, sv) \
  IOS_DISPATCH(dt, sv, 0); IOS_DISPATCH(dt, sv, 1); IOS_DISPATCH(dt, sv, 3); IOS_DISPATCH(dt, sv, 8); \
  IOS_DISPATCH(dt, sv, 9); IOS_DISPATCH(dt, sv, 11); IOS_DISPATCH(dt, sv, 15)
  IOS_DISPATCH_ALL(0, 1); IOS_DISPATCH_ALL(0, 0); IOS_DISPATCH_ALL(1, 1); IOS_DISPATCH_ALL(1, 0);
  IOS_DISPATCH(2, 1, 3); IOS_DISPATCH(2, 1, 15); IOS_DISPATCH(2, 0, 3); IOS_DISPATCH(2, 0, 15);
#undef IOS_DISPATCH_ALL
#undef IOS_DISPATCH
  return cudaErrorInvalidValue;
}

// the layout kernels store 8-channel vectors (16 B aligned) and index pixels in 32 bits
static bool layout_ok(const View& v, int N) {
  return v.C % 8 == 0 && v.cstride % 8 == 0 && v.coff % 8 == 0 && (v.ptr & 15) == 0 &&
         (int64_t)N * v.H * v.W * (v.C / 8) < (int64_t)INT_MAX;
}
static int layout_grid(int64_t npix) {
  const int64_t g = (npix + 255) / 256;
  return (int)(g < 148 * 8 ? (g > 0 ? g : 1) : 148 * 8);
}

cudaError_t launch_nchw_to_nhwc(const float* in, const View& out, int dtype, int N, int C, cudaStream_t st) {
  if (!layout_ok(out, N)) return cudaErrorInvalidValue;
  nchw_to_nhwc_kernel<<<layout_grid((int64_t)N * out.H * out.W * (out.C / 8)), 256, 0, st>>>(in, out, dtype, N, C);
  return cudaGetLastError();
}

cudaError_t launch_nchw_unfold(const float* in, const View& out, int dtype, int N, int C, int W, int kw, int sw, int pw,
                               cudaStream_t st) {
  if (!layout_ok(out, N)) return cudaErrorInvalidValue;
  nchw_unfold_kernel<<<layout_grid((int64_t)N * out.H * out.W * (out.C / 8)), 256, 0, st>>>(in, out, dtype, N, C, W, kw,
                                                                                            sw, pw);
  return cudaGetLastError();
}

cudaError_t launch_nhwc_to_nchw(const View& in, int dtype, float* out, int N, int C, cudaStream_t st) {
  const int64_t total = (int64_t)N * C * in.H * in.W;
  if (total >= (int64_t)INT_MAX) return cudaErrorInvalidValue;
  nhwc_to_nchw_kernel<<<layout_grid(total), 256, 0, st>>>(in, dtype, out, N, C);
  return cudaGetLastError();
}

cudaError_t launch_l2_flush(void* buf, int64_t bytes, cudaStream_t st) {
  l2_flush_kernel<<<148 * 4, 256, 0, st>>>(reinterpret_cast<int4*>(buf), bytes / 16);
  return cudaGetLastError();
}

}  // namespace ios
#endif  // !IOS_INST_DT
