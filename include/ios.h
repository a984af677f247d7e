/* ios.h — C-ABI of the B200-native IOS stage executor (arXiv 2011.01302).
 *
 * Citations: P:n = /root/reference/PAPER.md line n.
 *
 * The library implements the paper's problem statement (Sec. 3) and Algorithm 1
 * with a B200 execution engine:
 *   ios_graph_create / ios_add_op   build G = (V, E); edges are tensors
 *   ios_stage_latency               GenerateStage's measurement of one stage (S', T) (Alg. 1 L25/L27)
 *   ios_schedule_dp                 InterOperatorScheduler with pruning P(r, s) per block
 *   ios_run                         executes Q stage by stage
 *
 * Conventions (all functions):
 *   - Every call returns ios_status; IOS_OK = 0. No C++ exception crosses the ABI.
 *   - Out-parameters are written only on IOS_OK. ios_last_error() returns a thread-local message
 *     describing the last failure on the calling thread (valid until the next call on that thread).
 *   - Ownership: the library COPIES every host array passed in (weights, biases, add weights,
 *     schedule arrays) and owns every device buffer it allocates, except the caller's I/O
 *     pointers of ios_run / ios_op_output, which stay caller-owned.
 *   - Threading: a graph is single-owner; calls on one handle are not re-entrant. Different
 *     graphs (e.g. one per GPU) are independent.
 *   - Device memory is touched lazily: graph construction and ios_schedule_dp with a cost
 *     callback never initialise CUDA, so they run on machines without a GPU.
 *   - There is no CPU fallback: without a usable sm_100 device, device calls return IOS_ERR_CUDA.
 */
#ifndef IOS_H_
#define IOS_H_

#include <stdint.h>

#if defined(__GNUC__)
#define IOS_API __attribute__((visibility("default")))
#else
#define IOS_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ios_graph_s* ios_graph;       /* opaque; library-owned; free with ios_graph_destroy */
typedef struct ios_schedule_s* ios_schedule; /* opaque; library-owned; free with ios_schedule_destroy */

typedef enum {
  IOS_OK = 0,
  IOS_ERR_INVALID_ARG = 1,
  IOS_ERR_DANGLING_INPUT = 2, /* an input id does not name an existing op */
  IOS_ERR_SHAPE = 3,          /* shapes of the inputs are inconsistent with the op */
  IOS_ERR_BLOCK = 4,          /* edge from a later block, non-contiguous block, or > 64 ops in a block */
  IOS_ERR_NOT_MERGEABLE = 5,  /* operator merge requested for a set that cannot be merged */
  IOS_ERR_NOT_A_STAGE = 6,    /* ops not in one block, repeated, or not a valid stage */
  IOS_ERR_BAD_SCHEDULE = 7,   /* Q is not a valid sequence of endings */
  IOS_ERR_CUDA = 8,           /* CUDA runtime error or no usable sm_100 device */
  IOS_ERR_OOM = 9,
  IOS_ERR_KERNEL = 10,        /* in-kernel dependency wait timed out (deadlock guard) */
  IOS_ERR_UNSUPPORTED = 11    /* valid request the engine does not implement */
} ios_status;

typedef enum {
  IOS_MATH_TF32 = 0,      /* fp32 storage, tcgen05 kind::tf32 operands, fp32 accumulation */
  IOS_MATH_BF16 = 1,      /* bf16 storage, tcgen05 kind::f16 (bf16) operands, fp32 accumulation */
  IOS_MATH_FP32_SIMT = 2  /* fp32 storage, CUDA-core fp32 FMA (reference-precision path) */
} ios_math;

typedef enum { IOS_CONCURRENT = 0, IOS_MERGE = 1 } ios_strategy;   /* T_i */

typedef enum {             /* which strategies GenerateStage may use (Fig. 6) */
  IOS_BOTH = 0,            /* IOS-Both (the paper's IOS)                                 */
  IOS_MERGE_ONLY = 1,      /* IOS-Merge: multi-op stages must be merged                  */
  IOS_PARALLEL_ONLY = 2    /* IOS-Parallel: concurrent execution only                    */
} ios_strategy_set;

typedef enum {
  IOS_OP_CONV = 0,           /* Conv(-ReLU) unit: 1 input                                     */
  IOS_OP_SEPCONV = 1,        /* Relu-SepConv unit: n inputs summed with add_weights, ReLU,
                                depthwise kernel_h x kernel_w (stride, pad), pointwise to out_channels  */
  IOS_OP_MAXPOOL = 2,        /* 1 input, window kernel_h x kernel_w                                   */
  IOS_OP_AVGPOOL = 3,        /* 1 input; IOS_F_COUNT_INCLUDE_PAD selects the divisor                   */
  IOS_OP_GLOBAL_AVGPOOL = 4, /* 1 input -> [N, C, 1, 1]                                               */
  IOS_OP_ADD = 5,            /* n inputs of equal shape: sum_i add_weights[i] * x_i                   */
  IOS_OP_CONCAT = 6,         /* n inputs, concatenated along C in order                       */
  IOS_OP_IDENTITY = 7,       /* 1 input, copied                                                        */
  IOS_OP_LINEAR = 8          /* FC head: 1 input of spatial size 1x1; a 1x1 conv (Z18)                 */
} ios_op_kind;

enum {
  IOS_F_RELU_POST = 1,          /* ReLU after the op (conv, sepconv, linear)        */
  IOS_F_RELU_PRE = 2,           /* ReLU on the input (conv, global avgpool; implied for sepconv) */
  IOS_F_CEIL_MODE = 4,          /* pooling output size rounds up (torch rule)         */
  IOS_F_COUNT_INCLUDE_PAD = 8   /* avgpool divisor counts padding                     */
};

typedef struct {
  int32_t kind;           /* ios_op_kind */
  int32_t block;          /* block id: the DP runs per block; blocks must be contiguous
                             in insertion order and edges may only go to the same or a later block */
  int32_t out_channels;   /* conv/sepconv/linear: Cout; ignored (derived) for the other kinds      */
  int32_t kernel_h, kernel_w, stride_h, stride_w, pad_h, pad_w;
  int32_t flags;          /* IOS_F_* */
  const float* weight;    /* host fp32, COPIED. conv: [Cout][Cin][kh][kw]; sepconv: depthwise [C][kh][kw]
                             followed by pointwise [Cout][C]; linear: [Cout][Cin]; NULL otherwise   */
  const float* bias;      /* host fp32 [Cout] or NULL (= 0), COPIED                                 */
  const float* add_weights; /* host fp32 [n_inputs] or NULL (= 1.0) for ADD / SEPCONV, COPIED       */
} ios_op_desc;

typedef struct {
  int32_t warmup;    /* untimed launches before the first trial (default 10)            */
  int32_t trials;    /* timed trials; the median trial mean is returned (default 5)      */
  int32_t reps;      /* back-to-back launches per trial between two CUDA events (default 20) */
  int32_t l2_flush;  /* non-zero: write 2x the L2 size between trials                    */
} ios_profile_opts;   /* DESIGN.md Z15 */

/* ---- graph construction ------------------------------------------------------------------- */

/* Creates G with op 0 = the graph input, an NCHW tensor [batch, c, h, w]. `device` is the CUDA
 * ordinal later calls run on (not touched here). */
IOS_API ios_status ios_graph_create(int32_t batch, int32_t c, int32_t h, int32_t w, ios_math math,
                            int32_t device, ios_graph* out);

/* Appends one op. `inputs` are existing op ids (0 = graph input), so insertion order is a
 * topological order (the sequential schedule's order). Shapes are inferred; weights are
 * copied. Writes the new op id (1, 2, ...) to *out_op_id. */
IOS_API ios_status ios_add_op(ios_graph g, const ios_op_desc* d, const int32_t* inputs, int32_t n_inputs,
                      int32_t* out_op_id);

IOS_API ios_status ios_graph_num_ops(ios_graph g, int32_t* n_ops);   /* excludes the input op 0 */
IOS_API ios_status ios_op_shape(ios_graph g, int32_t op, int32_t shape_nchw[4]);
/* Block structure: the number of blocks, and for one block (by position) its ops in insertion order. */
IOS_API ios_status ios_graph_num_blocks(ios_graph g, int32_t* n_blocks);
IOS_API ios_status ios_graph_block_ops(ios_graph g, int32_t block_pos, int32_t* ops, int32_t cap, int32_t* n_ops,
                               int32_t* block_id);
/* 1 if the ops can be executed as one merged convolution (reading Z4), else 0. */
IOS_API ios_status ios_stage_mergeable(ios_graph g, const int32_t* ops, int32_t n_ops, int32_t* mergeable);

/* ---- measurement ---------------------------------------------------------------------------- */

/* Latency in ms of running the stage {ops} (one block) with strategy t on the device: its groups
 * (connected components) run concurrently inside ONE persistent launch, or the ops are
 * merged into one convolution. Inputs of the stage are taken from the graph's
 * activation buffers (synthetic contents). Synchronises. IOS_ERR_NOT_MERGEABLE for an illegal
 * merge (GenerateStage turns that into L_merge = inf, Alg. 1 L28-29). opts may be NULL. */
IOS_API ios_status ios_stage_latency(ios_graph g, const int32_t* ops, int32_t n_ops, ios_strategy t,
                             const ios_profile_opts* opts, double* out_ms);

/* ---- schedules ------------------------------------------------------------------------------ */

/* Stage cost for the DP: milliseconds, INFINITY = illegal. `stage_mask` bit i = the i-th op of
 * `block` in insertion order. Must be deterministic for bit-exact schedules. */
typedef double (*ios_cost_fn)(void* ctx, int32_t block, uint64_t stage_mask, ios_strategy t);

/* Algorithm 1 per block with pruning P(r, s) (r = max ops per group, s = max groups per stage;
 * r or s <= 0 means unbounded), block schedules concatenated in block order. cost = NULL
 * measures every distinct stage with ios_stage_latency (cached per (block, mask, T)).
 * Ending order and ties: DESIGN.md Z1/Z2. *out_cost_ms = left fold of the stage costs. */
IOS_API ios_status ios_schedule_dp(ios_graph g, int32_t r, int32_t s, ios_cost_fn cost, void* ctx,
                           ios_schedule* out, double* out_cost_ms);
/* Same with a strategy set (IOS-Both / IOS-Merge / IOS-Parallel) and optional search statistics
 * (out_stats may be NULL): [0] states, [1] transitions, [2] distinct stages costed. */
IOS_API ios_status ios_schedule_dp_ex(ios_graph g, int32_t r, int32_t s, ios_strategy_set set, ios_cost_fn cost,
                              void* ctx, ios_schedule* out, double* out_cost_ms, int64_t out_stats[3]);
/* Measured refinement (an engine extension beyond the paper): the device-profiled DP is run under a
 * small family of cost models -- pruning (r, s), (min(r,2), s), (1, s), each with every measured
 * stage latency biased by -beta_us, 0, +beta_us -- plus the greedy and sequential stages of every
 * block whose greedy stages lie in P(r, s) (other blocks keep the plain DP's stages); every
 * distinct candidate schedule is stage-tuned and run in context (ios_run_timeline, `reps` runs, L2
 * flushed), and each block keeps the candidate whose stages took the least in-run time there.
 * Every block of the result is a schedule in Algorithm 1's search space under pruning (r, s),
 * chosen by measurement. out_stats (may be NULL): [0..2] as ios_schedule_dp_ex for (r, s) unbiased,
 * [3] = candidates * 1000 + blocks taken from a candidate other than the plain DP. Synchronises. */
IOS_API ios_status ios_schedule_refine(ios_graph g, int32_t r, int32_t s, int32_t reps, double beta_us,
                                       ios_schedule* out, int64_t out_stats[4]);
IOS_API ios_status ios_schedule_sequential(ios_graph g, ios_schedule* out);  /* one op per stage   */
IOS_API ios_status ios_schedule_greedy(ios_graph g, ios_schedule* out);      /* all ready ops       */
/* Builds a schedule from explicit stages: stage i has stage_sizes[i] ops taken consecutively from
 * `ops`, with strategy strategies[i]. Validated (IOS_ERR_BAD_SCHEDULE / IOS_ERR_NOT_MERGEABLE). */
IOS_API ios_status ios_schedule_create(ios_graph g, int32_t n_stages, const int32_t* stage_sizes, const int32_t* ops,
                               const int32_t* strategies, ios_schedule* out);
IOS_API ios_status ios_schedule_num_stages(ios_schedule q, int32_t* n);
IOS_API ios_status ios_schedule_stage(ios_schedule q, int32_t i, int32_t* ops, int32_t cap, int32_t* n_ops,
                              ios_strategy* t, double* latency_ms);

/* Stage tuner (an extension beyond the paper: the tile decomposition of each stage, not the
 * schedule). Every stage of Q is measured on the device under each of the library's tiling
 * variants (split-K granularity) with the ios_stage_latency protocol (`trials` x a CUDA graph of
 * `reps` back-to-back launches, median; <= 0 = defaults 3 and 10) and later runs of ANY schedule
 * use the fastest variant for that stage. Does not change Q or its outputs beyond floating-point
 * summation order. Synchronises. Errors: IOS_ERR_INVALID_ARG, IOS_ERR_CUDA, IOS_ERR_KERNEL. */
IOS_API ios_status ios_schedule_tune(ios_graph g, ios_schedule q, int32_t trials, int32_t reps);
/* The tuner's per-stage choices as a text file (one "block_pos mask strategy variant" line per
 * stage), so another process replays exactly the plans that were timed (e.g. under a profiler).
 * Loading checks the graph (op count, batch, math) and touches the device. */
IOS_API ios_status ios_tile_variants_save(ios_graph g, const char* path);
IOS_API ios_status ios_tile_variants_load(ios_graph g, const char* path);

/* ---- execution ------------------------------------------------------------------------------ */

/* Runs Q on `d_input` (device, caller-owned, NCHW fp32 [batch, c, h, w] contiguous) and writes the
 * last op's output to `d_output` (device, caller-owned, NCHW fp32 contiguous). Stream-ordered and
 * asynchronous on `cuda_stream` (a cudaStream_t; NULL = legacy default stream). The first call for
 * a schedule builds its stage plans and captures them into a CUDA graph (re-captured after
 * ios_schedule_tune replaced a plan). IOS_ERR_KERNEL: a dependency wait of an EARLIER run on this
 * graph timed out (the flag is host-mapped and read at the next call; see ios_sync). */
IOS_API ios_status ios_run(ios_graph g, ios_schedule q, const void* d_input, void* d_output, void* cuda_stream);
/* Same with HOST buffers: copies the input in, runs, copies the output back, synchronises.
 * IOS_ERR_KERNEL if an in-kernel dependency wait of this run timed out (outputs invalid). */
IOS_API ios_status ios_run_host(ios_graph g, ios_schedule q, const float* h_input, float* h_output, void* cuda_stream);
/* Synchronises `cuda_stream` (and the library's own stream) and reports IOS_ERR_KERNEL if an
 * in-kernel dependency wait of any earlier run on this graph timed out (the ~4 s deadlock guard:
 * the outputs of that run are invalid). ios_run itself reports such a flag at its next call. */
IOS_API ios_status ios_sync(ios_graph g, void* cuda_stream);
/* Copies op `op`'s most recent output (NCHW fp32) to caller-owned device memory. */
IOS_API ios_status ios_op_output(ios_graph g, int32_t op, void* d_out, void* cuda_stream);
/* In-run stage timeline (the stage profiler "in context"): runs Q `reps` times exactly as ios_run
 * does (one CUDA graph, programmatic dependent launch between stages), each run after an L2 flush
 * if l2_flush != 0, with every stage launch stamping its CTAs' earliest start (after the PDL wait)
 * and latest exit on the device's global timer. Per stage i, stage_us[3i..3i+2] = mean over reps of
 * (start, end) in us relative to the first stage's start, and of the ATTRIBUTABLE time
 * end_i - end_{i-1} (stage 0: end - start; empty stages 0), which sums to the schedule's span.
 * d_input/d_output as ios_run (device, caller-owned). cap >= 3 * #stages. Synchronises. */
IOS_API ios_status ios_run_timeline(ios_graph g, ios_schedule q, const void* d_input, void* d_output, int32_t reps,
                                    int32_t l2_flush, double* stage_us, int32_t cap);
/* Number of kernel launches one ios_run of q performs (stage kernels + boundary layout kernels). */
IOS_API ios_status ios_schedule_launches(ios_graph g, ios_schedule q, int32_t* n_launches);

/* Diagnostic timeline of ONE launch of a stage: per CTA 16 uint64 stamps (0 = not reached): slot 0
 * = %globaltimer ns at the CTA's entry, slots 1-15 = SM clock cycles since that entry, plus 1:
 * 1 prologue done, 2 first A chunk issued, 3 producer done, 4 MMA done, 5 first accumulator ready,
 * 6 epilogue/SIMT done, 7 teardown, 8 exit, 9-15 path-specific. out must hold grid*16. */
IOS_API ios_status ios_stage_trace(ios_graph g, const int32_t* ops, int32_t n_ops, ios_strategy t, uint64_t* out,
                                   int32_t cap, int32_t* grid);

/* ---- stage-latency cache (checkpoint / resume of long searches) ------------------------------ */
IOS_API ios_status ios_latency_cache_save(ios_graph g, const char* path);
IOS_API ios_status ios_latency_cache_load(ios_graph g, const char* path);
/* Checkpoint the cache to `path` after every block the device-profiled DP finishes measuring, so a
 * long search (NASNet, RandWire) resumes with ios_latency_cache_load; NULL or "" turns it off. */
IOS_API ios_status ios_latency_cache_autosave(ios_graph g, const char* path);

IOS_API const char* ios_last_error(void);
/* Content hash of the sources this library was compiled from (build.py), for provenance checks. */
IOS_API const char* ios_build_id(void);
IOS_API void ios_schedule_destroy(ios_schedule q);
IOS_API void ios_graph_destroy(ios_graph g);

#ifdef __cplusplus
}
#endif
#endif /* IOS_H_ */
