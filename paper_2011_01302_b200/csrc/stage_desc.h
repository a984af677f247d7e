// Device-visible descriptors of one stage plan.
// Plain structs shared by the host planner (plan.cpp) and the persistent stage kernel
// (stage_kernel.cu). One stage = one launch; the kernel walks a tile list that spans every
// member op of the stage ("problems"), in an order where every dependency points backwards.
#pragma once
#include <stdint.h>

namespace ios {

// ---- tile geometry -----------------------------------------------------------------------------
constexpr int kBM = 128;                  // GEMM tile rows (output pixels); UMMA M = 128, cta_group::1
constexpr int kChunkBytes = 128;          // bytes of K per pipeline stage (32 fp32 / 64 bf16 elements)
constexpr int kStages = 4;                // ring depth at the widest tile (BN = 256): 4 x 48 KB
constexpr int kMaxBN = 256;               // UMMA N <= 256
constexpr int kAStageBytes = kBM * kChunkBytes;         // 16 KB
constexpr int kBStageBytes = kMaxBN * kChunkBytes;      // 32 KB
constexpr int kRingBytes = kStages * (kAStageBytes + kBStageBytes);   // 192 KB of ring slots
constexpr int kMaxSlots = 16;             // deepest ring (narrow tiles: slot = 16 KB A + BN x 128 B)
constexpr int kBarBytes = 512;            // mbarriers, TMEM slot, flags
constexpr int kBiasBytes = 2 * kMaxBN * 4; // bias slice per accumulator buffer
constexpr int kDescBytes = 14 * 1024;     // stage descriptor table (problems | views | segments) copy
constexpr int kEpiBytes = 4 * 4096;       // epilogue staging: 32 rows x 128 B per epilogue warp
constexpr int kSmemBytes = kRingBytes + kBarBytes + kBiasBytes + kDescBytes + kEpiBytes;
constexpr int kProducerWarps = 4;         // warps 0-3: A gather (cp.async) + B bulk copy
constexpr int kEpilogueWarp0 = 4;         // warps 4-7: TMEM -> registers -> global; SIMT tiles
constexpr int kMmaWarp = 8;               // warp 8: tcgen05.mma issuer + TMEM allocator
constexpr int kThreads = 9 * 32;
constexpr int kTmemCols = 512;            // 2 accumulator buffers x 256 columns
constexpr int kMaxProblems = 96;
constexpr int kCounterBase = 2;       // counters[0..1]: the 64-bit launch counter
constexpr int kSlabSplits = 1;            // split-K: problems with <= this many splits store per-split
                                          // slabs summed in split order (deterministic); the others reduce
                                          // into one zeroed slab (red.add: measured faster at every split
                                          // count, so the default is 1 = always reduce; IOS_SLAB_SPLITS=32
                                          // is the deterministic mode)
constexpr int kMaxSegs = 8;               // merged conv: one output segment per branch

enum ProblemKind : int32_t {
  PK_GEMM = 0,      // implicit-GEMM conv / merged conv / pointwise / linear on tcgen05
  PK_MAXPOOL = 1,
  PK_AVGPOOL = 2,
  PK_GAVGPOOL = 3,
  PK_ADD = 4,       // sum_i w_i x_i
  PK_COPY = 5,      // concat (non-elided) / identity: gather input channel ranges into the output
  PK_DWCONV = 6,    // sepconv front half: ReLU(sum_i w_i x_i) -> depthwise k x k
};

// ET_F32: fp32 storage rounded to TF32 (tcgen05 kind::tf32); ET_F32X: exact fp32, CUDA-core FMA GEMM
enum ElemType : int32_t { ET_F32 = 0, ET_BF16 = 1, ET_F32X = 2 };

// An NHWC activation view: element (n, h, w, c) at ptr + ((n*H + h)*W + w)*cstride + coff + c.
// C is the padded channel count (multiple of 8); channels [Cl, C) hold zeros.
struct View {
  uint64_t ptr;
  int32_t cstride, coff, C, Cl, H, W;   // C = padded channels, Cl = logical channels
};

struct Segment {           // output columns [n0, n1) of a GEMM go to `out` at channel n - n0
  int32_t n0, n1;
  View out;
  int32_t relu, pad_;
};

// x / d for 0 <= x < 2^31 with one multiply-high (round-up multiplier method); built on the host.
struct FastDiv {
  uint32_t d, mul, shift, pad_;
};
inline FastDiv make_fastdiv(uint32_t d) {
  uint32_t sh = 0;
  while ((1ull << sh) < d) ++sh;
  const uint64_t mul = ((1ull << 32) * ((1ull << sh) - d)) / d + 1;
  return FastDiv{d, (uint32_t)mul, sh, 0};
}

// Row-band dependency of a stage member on an in-stage producer: instead of waiting
// for every tile of the producer, a consumer tile waits only for the producer tiles ("bands") that
// cover the input rows it reads. Rows are global rows g = n * H + h of the producer's output.
struct DepBand {
  int32_t mode;      // 0: whole producer (dep_idx / dep_target); 1: dense GEMM M tiles of bsz pixels;
                     // 2: patch M tiles (tN images x tR rows x tiles_w column tiles); 3: SIMT tiles of
                     // bsz pixel items; 4: SIMT tiles of bsz quad items, tiles_w = quads per row
  int32_t ctr;       // counter index of band 0 (counters[ctr + b] += 1 per unit finishing band b)
  int32_t target;    // units per band per launch (GEMM: n tiles x splits; SIMT: 1)
  int32_t bsz, H, W, tN, tR, tiles_h, tiles_w, nbands, pad_;
};

struct Problem {
  int32_t kind, dtype;
  int32_t tile_begin, n_tiles;      // tiles [tile_begin, tile_begin + n_tiles) of the stage
  int32_t done_idx;                 // counters[done_idx] += 1 per finished output tile
  int32_t n_deps;
  int32_t dep_idx[6];               // wait until counters[dep_idx[i]] >= dep_target[i]
  int32_t dep_target[6];
  int32_t band_begin;               // DepBand entries [band_begin, band_begin + n_deps) (-1: whole waits)
  int32_t band_ctr;                 // this problem's own bands: counters[band_ctr + band] (-1: none)
  int32_t batch, flags;             // flags: IOS_F_* of the op
  int32_t kh, kw, sh, sw, ph, pw;
  int32_t Ho, Wo;
  int32_t in_begin, n_in;           // views[in_begin .. in_begin + n_in)
  View out;                         // SIMT output / GEMM: unused (segments)
  uint64_t wts;                     // GEMM: packed weights; DWCONV: fp32 tap-major [kh*kw][C]
  uint64_t bias;                    // fp32 [N padded]
  uint64_t add_w;                   // fp32 [n_in] or 0
  // GEMM geometry
  int32_t M, K, k_chunks;           // M = batch*Ho*Wo, K = kh*kw*Cin_p (elements)
  int32_t BN, n_tiles_n, m_tiles;   // tile = (m, n, split)
  int32_t split, chunks_per_split;
  int32_t Npad8;                    // packed weight rows (multiple of 8)
  int32_t seg_begin, n_seg;
  uint64_t workspace;               // split-K fp32 partials, per output tile [split][kBM][BN] (swap-AB:
                                    // channel-major [split][128][BN]), summed in split order; with more
                                    // than kSlabSplits splits one zeroed [kBM][BN] slab that the splits
                                    // reduce into (red.add) and the finalize re-zeroes
  int32_t tilectr_idx;              // split-K arrival counters base
  int32_t slabs;                    // split-K: 1 per-split slabs, 0 one reduction slab (see workspace)
  int32_t signal;                   // 1: a later member of the stage waits on done_idx (or on its bands)
  FastDiv fd_howo, fd_wo, fd_split, fd_ntn, fd_cin, fd_kw;   // divisors of the tile / im2col decode
  // SIMT geometry
  int32_t items_per_tile, n_items;  // items = output pixels (x channel vectors handled inside)
  int32_t dwq;                      // window ops (dw / max / avg, square k in {3,5,7}, stride 1-2):
                                    // items are quads of dwq horizontally adjacent output pixels
                                    // sharing one loaded input row span (0 = one pixel per item)
  int32_t a_tma;                    // 1: the activation operand is a plain [M, C] matrix loaded by TMA
  int32_t swap_ab;                  // 1: weights are the MMA A operand (128 output channels per tile),
                                    //    the M (<= 128) pixels are MMA N = BN; m_tiles count channel tiles
  int32_t tt;                       // 1: "tap TMA" im2col: per K chunk (tap, 32/64-channel block) one 4D
                                    //    tensor TMA of a (tN images x tR rows x tWt cols) output patch;
                                    //    M tiles are such patches (tile row r = (nn*tR + i)*tWt + j);
                                    //    K = taps x kblk channel blocks (zero-padded)
  int32_t kblk, tN, tR, tWt, tiles_h, tiles_w;
  FastDiv fd_kblk, fd_thw, fd_tw, fd_tilw, fd_tilh;
  uint64_t tmap_a;                  // global address of its CUtensorMap (2D / 4D tiled, 128B swizzle)
  // fused Relu-SepConv: the producer warps compute the depthwise half of the unit
  // straight into the A operand of its pointwise GEMM (patch M tiles as with tap TMA, K = the
  // input channels); inputs [in_begin, in_begin + n_in) are aggregated with add_w first
  int32_t fdw;                      // 1: fused depthwise A producer
  int32_t dk, ds, dp;               // depthwise window (square k in {3, 5, 7}), stride, padding
  int32_t dH, dW;                   // depthwise input spatial size
  uint64_t dww;                     // fp32 tap-major [k*k][Cin_p] depthwise weights
  uint64_t dwc;                     // fp32 chunk-major [k_chunks][k*k][elems per 128 B chunk] (halo path)
  int32_t hws, hhs;                 // halo path: input window of one patch tile = hhs rows x hws columns,
                                    // staged by ONE 4D tensor TMA (tmap_a) per K chunk, OOB = padding zeros
  // cluster split-K (F_CSK): the split index s = g * csplit + r; the csplit splits of one output tile
  // run on csplit CTAs of one thread-block cluster (tiles laid out so that r == cluster rank % csplit)
  // and are summed through distributed shared memory: CTA rank r owns tile rows
  // [r * 128 / csplit, (r + 1) * 128 / csplit); the others push their fp32 partial rows into its
  // receive buffer (st.async + mbarrier complete_tx). With split == csplit that is the whole
  // reduction; with more (split / csplit global groups) the owners' csplit-summed rows go through the
  // global red.add + rendezvous path. 1 = no cluster reduction.
  int32_t csplit, csk_pad_;
  FastDiv fd_q4;                    // split-K finalize: divisor BN / 4 (column quads per tile row)
};

// Kernel feature classes: the stage kernel is instantiated per class with only the code paths its
// stages use (measured: the unused paths' code and registers cost 7-10 % end to end through
// instruction-cache misses and spills). The host picks the smallest class covering a stage.
enum KernelFeature : int32_t {
  F_GATHER = 1,   // implicit-im2col cp.async producer (pre-ReLU convs, narrow / unaligned inputs)
  F_FDW = 2,      // fused Relu-SepConv producers (halo + register forms)
  F_TRACE = 4,    // per-CTA %globaltimer timeline (ios_stage_trace)
  F_CSK = 8,      // cluster split-K (Problem.csplit > 1): clusters of kClusterCtas CTAs, DSMEM reduction
};
constexpr int kFeatLean = 0, kFeatGather = F_GATHER, kFeatFull = F_GATHER | F_FDW,
              kFeatTrace = kFeatFull | F_TRACE | F_CSK;
constexpr int kClusterCtas = 4;   // cluster size of F_CSK launches (csplit in {2, 4})

// halo path (single-input fused Relu-SepConv): the stage runs its smem ring with 3 slots; slot 3's
// B region holds the input window of the chunk, slot 3's A region the chunk's depthwise weights
constexpr int kHaloBytes = kBStageBytes;          // 32 KB: <= 256 pixels x 128 B
constexpr int kHaloWBytes = kAStageBytes;         // 16 KB: k*k x 128 B (fp32) / 256 B (bf16 chunk)

struct StageDesc {
  uint64_t problems;                // Problem[n_problems]
  uint64_t views;                   // View[]
  uint64_t segs;                    // Segment[]
  uint64_t counters;                // int32[n_counters]; [0..1] = 64-bit launch counter (see uses_counters)
  uint64_t err;                     // int32 error flag (dependency-wait timeout), host-mapped pinned memory
  uint64_t trace;                   // optional uint64 [grid][16] timeline (0 = off)
  uint64_t stamp;                   // optional uint64 [2]: atomicMin of the CTAs' start (after the
                                    // PDL wait) and atomicMax of their exit, %globaltimer ns (0 = off)
  int32_t n_problems, n_tiles, n_counters, has_gemm;
  int32_t blob_bytes;               // problems | views | segments, contiguous from `problems`
  int32_t views_off, segs_off, bands_off;
  int32_t uses_counters;            // any in-stage dependency or split-K: counters[0..1] count launches
                                    // (epoch), the others grow monotonically (targets epoch-relative,
                                    // compared wrap-safely mod 2^32)
  int32_t feat;                     // KernelFeature bits this stage needs (host: picks the instantiation)
  int32_t slot_bytes;               // ring slot stride: A region (16 KB: 128 rows x 128 B) then the B region
                                    // (the stage's widest B operand, BN rows x 128 B, rounded to 1 KB);
                                    // narrow tiles get a deeper ring (more bytes in flight per CTA)
  int32_t ring_slots;               // smem ring depth this launch (<= kMaxSlots), or 3 x 48 KB when a halo
                                    // problem borrows the last slot
  int32_t cluster;                  // 1, or kClusterCtas: the launch is a cluster launch (F_CSK)
  int32_t rbuf_off;                 // F_CSK: receive buffer at smem ring + rbuf_off (end of the ring region)
  int32_t rbuf_stride;              // F_CSK: bytes per received row (the widest csplit problem's BN x 4 + 16)
  int32_t pad_;
};

}  // namespace ios
