/*
 * tp_b200.h — C ABI of the B200-native multi-dimensional tensor-parallel linear layer.
 *
 * The operation (PAPER.md = P:Lnnn, SPEC.md = S:Lnnn; DESIGN.md lists every reading):
 *   Y = alpha * X . W + b,  dX = alpha * dY . W^T,  dW = alpha * X^T . dY,  db = 1^T dY
 * with X [M,K], W [K,N], Y [M,N] row-major (reading A1), partitioned over
 * p GPUs in one of four modes:
 *   TP_1D    Megatron column / row split
 *   TP_2D    SUMMA on a q x q grid, p = q^2
 *   TP_2P5D  q x q x d grid, depth d given by the user, p = d q^2
 *   TP_3D    l x l x l cube, p = l^3
 * Grid constraints P:L530; no silent fallback to 1D.
 *
 * Conventions for every entry point:
 *   - Pointers named x, w, y, dy, dx, dw, bias, dbias, saved, ws, A, B, C, D, dst,
 *     global, shard are DEVICE pointers on the grid's CUDA device, owned by the
 *     caller; the library never frees them. Host pointers appear only where noted.
 *   - Shards are dense row-major blocks: a tensor's local block of extent
 *     (rows, cols) (see tp_shard_extent) is stored with row stride = cols elements.
 *   - dtype TP_BF16: operands and outputs bf16, fp32 accumulate (tcgen05/TMEM);
 *     TP_FP32: everything fp32 (SIMT FFMA path). Bias has the operand dtype.
 *   - `stream` is a cudaStream_t passed as void*. Work is stream-ordered: it
 *     starts after prior work on `stream` and later work on `stream` sees the
 *     results. No host synchronisation, EXCEPT with TP_TRANSPORT_LOCAL, whose
 *     collectives rendezvous on the host (each rank must be on its own thread).
 *   - Every argument check runs on the host BEFORE anything is enqueued. On error
 *     nothing is enqueued, the status says which class, tp_last_error() (thread-
 *     local) says why.
 *   - Collective contract (like NCCL): every rank of a grid calls tp_linear_fwd /
 *     tp_linear_bwd with an identical descriptor, in the same order.
 */
#ifndef TP_B200_H
#define TP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  TP_OK = 0,
  TP_ERR_CONSTRAINT = 1,  /* world does not factor as the mode requires */
  TP_ERR_INDIVISIBLE = 2, /* a dim is not divisible by the mode's split */
  TP_ERR_SHAPE = 3,       /* bad shape / alignment (TMA needs 16-byte row strides and bases) */
  TP_ERR_ARG = 4,         /* null / out-of-range argument */
  TP_ERR_CUDA = 5,        /* a CUDA runtime call failed */
  TP_ERR_NCCL = 6,        /* an NCCL call failed */
  TP_ERR_WORKSPACE = 7,   /* ws_bytes smaller than tp_workspace_size() */
  TP_ERR_UNSUPPORTED = 8  /* valid request this build does not implement */
} tp_status;

typedef enum { TP_1D = 1, TP_2D = 2, TP_2P5D = 3, TP_3D = 4 } tp_mode;
typedef enum { TP_BF16 = 0, TP_FP32 = 1 } tp_dtype;

/* How ranks talk.
 *   NCCL  one process (or thread) per GPU; id128 = ncclUniqueId from rank 0's
 *         tp_get_unique_id, broadcast by the caller (e.g. torch.distributed).
 *         Per-axis communicators come from ncclCommSplit.
 *   LOCAL all ranks in ONE process, one host thread per rank, any devices
 *         (several ranks may share a device). Collectives are stream-ordered
 *         device copies / reduction kernels between the ranks' buffers, after a
 *         host rendezvous. Used to run multi-rank grids on a single GPU.
 *   NONE  no communication: grid planning (extents, workspace) for any world,
 *         compute only when world == 1. */
typedef enum { TP_TRANSPORT_NCCL = 0, TP_TRANSPORT_LOCAL = 1, TP_TRANSPORT_NONE = 2 } tp_transport;

typedef enum { TP_TENSOR_X = 0, TP_TENSOR_W = 1, TP_TENSOR_Y = 2, TP_TENSOR_BIAS = 3 } tp_tensor;

/* tp_linear_desc.flags */
#define TP_FLAG_W25_DEPTH_SHARDED 0x1u /* 2.5D: W also split over depth (1/p at rest); AG in fwd, RS of dW */
#define TP_FLAG_SERIAL 0x2u            /* debug: run collectives on the compute stream (no overlap) */
/* Y = gelu(alpha X.W + b) (exact erf form; oracle/activation.py): the
 * forward keeps the pre-activation Z (the Y shard) in `saved` after the mode's own content and
 * tp_linear_bwd takes dL/dY, forming dZ = dY * gelu'(Z) in `ws` (tp_workspace_size counts both). */
#define TP_FLAG_GELU 0x8u
/* 2D / 2.5D forward with Cannon's algorithm ("SUMMA and Cannon"; skew + unit cyclic
 * shifts along the grid rows / columns) instead of SUMMA's broadcasts; same layouts and
 * results. The backward keeps the SUMMA ABT / ATB schedule. */
#define TP_FLAG_CANNON 0x10u
/* 2.5D as Solomonik & Demmel's 2.5D matrix multiplication (P:L526 cites it; SURVEY 8(f)
 * NEXT-4; oracle/solomonik.py, reading N5) instead of the paper's batch-split 2.5D: every
 * layer holds the full q x q block layout (X [M/q, K/q], W [K/q, N/q], Y [M/q, N/q] at
 * (dep, i, j), replicated over depth), layer dep runs the SUMMA steps [dep q/d, (dep+1) q/d),
 * Y is all-reduced over depth, dX / dW are depth-broadcast from the layer that reduced them.
 * Needs q % d == 0 and M, K, N divisible by q; excludes TP_FLAG_W25_DEPTH_SHARDED, CANNON
 * and PEER_FUSED (TP_ERR_ARG). */
#define TP_FLAG_SOLOMONIK 0x20u

typedef struct tp_grid tp_grid; /* opaque; library-owned (communicators, streams, events) */

typedef struct {
  int64_t M, K, N;   /* GLOBAL shape: X [M,K], W [K,N], Y [M,N] */
  tp_dtype dtype;
  int split_1d;      /* TP_1D only: 0 = column-parallel (W split by columns), 1 = row-parallel */
  int parity_3d;     /* TP_3D only: 0 or 1; parity 1 swaps axes b and c so Y(0) == X(1) layout */
  uint32_t flags;    /* TP_FLAG_* */
  float alpha;       /* Y = alpha * X.W + b */
} tp_linear_desc;

/* ---- errors ------------------------------------------------------------------------- */
const char* tp_status_string(tp_status s);
/* Detail of the last error on the calling thread ("" if none). Valid until the next call. */
const char* tp_last_error(void);
/* Library version string, and the CUDA arch it was built for ("sm_100a"). */
const char* tp_version(void);

/* ---- grid (P:L287 parallel context) ---------------------- */
/* Writes a 128-byte rendezvous id into id128 (host memory, 128 bytes).
 * NCCL: ncclGetUniqueId (call on ONE rank, share the bytes). LOCAL: a fresh
 * process-unique tag naming an in-process world. NONE: zeros. */
tp_status tp_get_unique_id(tp_transport transport, void* id128);

/* Creates this rank's view of the grid and its per-axis communicators.
 *   mode   TP_1D .. TP_3D;  world = p;  rank in [0, p)
 *   q      side: 2D j, 2.5D k, 3D l; pass 0 to derive it from world (and d)
 *   d      2.5D depth (>= 1); ignored (treated as 1) by other modes
 *   cuda_device  the GPU of this rank
 *   id128  host pointer to the id from tp_get_unique_id (unused for NONE)
 * Coordinates are row-major: 1D (r); 2D rank = i q + j; 2.5D rank = dep q^2 + i q + j
 * (depth outermost); 3D rank = a l^2 + b l + c. Groups along an axis list
 * their members by ascending coordinate.
 * Errors: TP_ERR_CONSTRAINT if world does not factor; TP_ERR_ARG; TP_ERR_NCCL/CUDA.
 * NCCL/LOCAL init is collective: all ranks of the world must call it. */
tp_status tp_grid_init(tp_grid** grid, tp_mode mode, int world, int rank, int q, int d,
                       int cuda_device, tp_transport transport, const void* id128);

/* coords[0..2]: 1D (r,0,0); 2D (i,j,0); 2.5D (dep,i,j); 3D (a,b,c). */
tp_status tp_grid_coords(const tp_grid* grid, int coords[3]);
/* dims[0..2] of the grid (unused = 1) and the number of axes. */
tp_status tp_grid_dims(const tp_grid* grid, int dims[3], int* ndims);
/* Members (global ranks, ascending coordinate) of this rank's line along `axis`;
 * members must hold dims[axis] ints. */
tp_status tp_grid_group(const tp_grid* grid, int axis, int* members);
tp_status tp_grid_destroy(tp_grid* grid);

/* Collective-contract check (debug; SURVEY 8(b) "Every rank of the grid must call fwd/bwd with
 * an identical desc, in the same order ... A debug flag verifies this"). When enabled, every
 * collective entry point (tp_linear_fwd/bwd, tp_layernorm_fwd/bwd, tp_rsa_fwd/bwd,
 * tp_attention_fwd/bwd) first exchanges a 64-bit hash of (entry point, per-grid call number,
 * desc fields, the entry point's scalar arguments) with every rank of the grid on the host and
 * returns TP_ERR_ARG - with nothing enqueued, on every rank - if any rank's hash differs, so a
 * mismatched call fails instead of deadlocking inside a collective. The exchange is a host
 * rendezvous (LOCAL) or a blocking 8-byte NCCL all-gather (NCCL): not stream-capturable, debug
 * only. A rank that skips the call entirely still hangs its peers. No effect at world == 1.
 * Collective when the grid is shared: every rank must set the same value. */
tp_status tp_grid_set_contract_check(tp_grid* grid, int enable);

/* Tuning knobs: every kernel-variant / dispatch choice the library does not derive from the
 * problem itself (GEMM kernel and tile forcing, split-K, raster, wide tiles, PDL, fused
 * attention, comm SM reservation). Defaults are the measured choices; a TP_* environment
 * variable of the same name, read once, overrides the default; tp_knob_set overrides both for
 * later calls (process-wide). tp_knobs writes a JSON array of {name, value, default, source
 * ("default" | "env" | "api"), what} into buf (NUL-terminated, truncated to cap; *needed =
 * required size). Errors: TP_ERR_ARG for an unknown name. */
tp_status tp_knob_set(const char* name, int value);
tp_status tp_knob_get(const char* name, int* value);
tp_status tp_knobs(char* buf, size_t cap, size_t* needed);

/* Failure detection. tp_grid_check: TP_OK, or TP_ERR_NCCL with the detail when a
 * communicator of the grid reports an asynchronous error (ncclCommGetAsyncError: a peer died,
 * a network / NVLink fault); non-blocking, callable from a watchdog thread while collectives
 * run. tp_grid_abort: aborts every communicator (ncclCommAbort), so collectives blocked on a
 * dead peer return; afterwards the grid only supports tp_grid_destroy. LOCAL / NONE: no-ops. */
tp_status tp_grid_check(const tp_grid* grid);
tp_status tp_grid_abort(tp_grid* grid);

/* ---- the grid's line communicators ("only incur communication on a sub-group") ---- */
/* One collective over this rank's line along `axis` (members by ascending coordinate, as
 * tp_grid_group), the primitive the schedules are built from:
 *   TP_COLL_BCAST          recv (in place) := recv of member `arg` (root position on the line)
 *   TP_COLL_REDUCE         recv := sum over members of send, significant at member `arg`
 *   TP_COLL_ALLREDUCE      recv := sum over members of send
 *   TP_COLL_ALLGATHER      recv [size*count] := concat over members of send [count]
 *   TP_COLL_REDUCESCATTER  recv [count] := slice `pos` of sum over members of send [size*count]
 *   TP_COLL_SHIFT          recv := send of member (pos + arg) mod size
 * count in elements of dt (TP_BF16 / TP_FP32), device buffers, stream-ordered on `stream`.
 * Collective: every member of the line calls it with the same op, count, dt and arg. A
 * size-1 line is the identity (NCCL: a 1-rank communicator, so the NCCL calls still run).
 * Errors: TP_ERR_ARG (axis, op, null buffers), TP_ERR_NCCL / TP_ERR_CUDA. */
typedef enum {
  TP_COLL_BCAST = 0, TP_COLL_REDUCE = 1, TP_COLL_ALLREDUCE = 2, TP_COLL_ALLGATHER = 3,
  TP_COLL_REDUCESCATTER = 4, TP_COLL_SHIFT = 5
} tp_collective;
tp_status tp_axis_collective(tp_grid* grid, int axis, tp_collective op, const void* send,
                             void* recv, size_t count, tp_dtype dt, int arg, void* stream);

/* ---- layout (P:L524 2D, P:L526 2.5D, P:L528 3D, P:L486-488 1D) ----------------------- */
/* Global block of `tensor` held by this rank: rows [row0, row0+rows), cols [col0, col0+cols).
 * BIAS is a [1, N] row. Gradients share their tensor's extent (dX~X, dW~W, dY~Y, db~BIAS).
 * Errors: TP_ERR_INDIVISIBLE (no padding), TP_ERR_ARG. Host only. */
tp_status tp_shard_extent(const tp_grid* grid, const tp_linear_desc* desc, tp_tensor tensor,
                          int64_t* row0, int64_t* rows, int64_t* col0, int64_t* cols);

/* Device bytes the caller must provide: ws (scratch, reusable after the call's work
 * completes on `stream`) and saved (written by fwd, read by the matching bwd: the 3D
 * gathered X and W, the 2.5D depth-gathered W). Either may be 0. The same ws size
 * serves fwd and bwd. Host only. */
tp_status tp_workspace_size(const tp_grid* grid, const tp_linear_desc* desc, size_t* ws_bytes,
                            size_t* saved_bytes);

/* ---- the hot path --------------------------------------------------------------------- */
/* Forward. x, w: this rank's shards; bias: this rank's bias shard or NULL; y: output
 * shard (written); saved: saved_bytes of device memory (NULL iff saved_bytes == 0);
 * ws: ws_bytes >= tp_workspace_size. Computes Y = alpha X.W + b in the mode's layout. */
tp_status tp_linear_fwd(tp_grid* grid, const tp_linear_desc* desc, const void* x, const void* w,
                        const void* bias, void* y, void* saved, void* ws, size_t ws_bytes,
                        void* stream);

/* Backward of the forward that wrote `saved`. dy: this rank's dY shard (Y's layout).
 * Writes dx (X's layout; may be NULL to skip), dw (W's layout), dbias (bias layout;
 * NULL to skip). x, w: the same shards given to fwd. */
tp_status tp_linear_bwd(tp_grid* grid, const tp_linear_desc* desc, const void* dy, const void* x,
                        const void* w, const void* saved, void* dx, void* dw, void* dbias,
                        void* ws, size_t ws_bytes, void* stream);

/* Model-boundary split/gather: copy this rank's block of the dense
 * row-major global tensor (device) into `shard`, or back. Bit-exact copies. */
tp_status tp_pack(const tp_grid* grid, const tp_linear_desc* desc, tp_tensor tensor,
                  const void* global, void* shard, void* stream);
tp_status tp_unpack(const tp_grid* grid, const tp_linear_desc* desc, tp_tensor tensor,
                    const void* shard, void* global, void* stream);

/* ---- fused peer-memory path ----------------------------------------- */
/* Registers a SYMMETRIC buffer: every rank of the grid calls this collectively, in the same
 * order, with its own copy of the same logical buffer (same size). Afterwards, for a pointer
 * p inside the buffer at offset o, the library can address every rank's p + o directly: raw
 * pointers for ranks of the same process (TP_TRANSPORT_LOCAL), CUDA IPC mappings across
 * processes (TP_TRANSPORT_NCCL, NVLink peer access). With TP_FLAG_PEER_FUSED, a 2D / 2.5D
 * layer whose x, w (and dy) shards lie in registered buffers at the same offsets on all ranks
 * runs as panel GEMMs that read the peers' shards with TMA (no broadcast, no reduce).
 * The buffer must stay allocated until tp_deregister_all / tp_grid_destroy. */
tp_status tp_register_buffer(tp_grid* grid, void* ptr, size_t bytes);
tp_status tp_deregister_all(tp_grid* grid);
#define TP_FLAG_PEER_FUSED 0x4u /* tp_linear_desc.flags: fused owner-computes panel GEMMs (2D, 2.5D, 3D l=2) */
/* With TP_FLAG_PEER_FUSED: every panel a rank reads from a peer is first pulled ONCE into local
 * workspace by the copy engine (cudaMemcpyAsync on the comm stream, after the grid barrier that
 * marks the owners' shards ready), and the panel GEMM reads the local copy. A panel GEMM that
 * reads a peer's shard directly re-reads it once per output tile row / column it feeds (~M/256
 * or N/256 times over NVLink); staged, each remote byte crosses the link exactly once - the same
 * bytes SUMMA receives. Staging is automatic for peers on another GPU; this flag forces it for
 * every peer (in-process ranks on one GPU: tests). */
#define TP_FLAG_PEER_STAGED 0x40u
/* Cumulative bytes this rank has pulled from peers by staging copies (host counter). */
tp_status tp_peer_staged_bytes(const tp_grid* grid, uint64_t* bytes);

/* ---- kernels exposed for parity tests and benchmarks ----------------------------------- */
/* Local GEMM, the per-step shard product of every mode:
 *   D[M,N] = alpha * (op(A) . op(B) + C) + bias[col]
 * op(A) = A [M,K] row-major (lda >= K) if trans_a == 0, else A is stored [K,M] (lda >= M);
 * op(B) = B [K,N] row-major (ldb >= N) if trans_b == 0, else B is stored [N,K] (ldb >= K).
 * C: fp32 [M,N] (ldc) or NULL; bias: in_dtype [N] or NULL; D: out_dtype, ldd.
 * TP_BF16 inputs run the tcgen05/TMEM/TMA kernels (bf16 x bf16 -> fp32; CTA-pair
 * cta_group::2 tiles when M > 128), TP_FP32 inputs the SIMT fp32 kernel. bf16 operands need
 * lda, ldb multiples of 8 and 16-byte aligned bases (TMA), else TP_ERR_SHAPE. D may alias C
 * (in-place accumulate). ws: optional device scratch (ws_bytes >= tp_gemm_ws_bytes() enables
 * split-K for grids with fewer tiles than SM pairs); NULL/0 disables split-K. */
tp_status tp_gemm(int trans_a, int trans_b, int64_t M, int64_t N, int64_t K, tp_dtype in_dtype,
                  const void* A, int64_t lda, const void* B, int64_t ldb, const float* C,
                  int64_t ldc, void* D, int64_t ldd, tp_dtype out_dtype, float alpha,
                  const void* bias, void* ws, size_t ws_bytes, void* stream);
/* Scratch bytes that enable split-K in tp_gemm for any shape. */
size_t tp_gemm_ws_bytes(void);

/* db = 1^T dY: column sums of a [rows, cols] row-major matrix (ld), fp32 accumulate. */
tp_status tp_colsum(const void* src, int64_t rows, int64_t cols, int64_t ld, tp_dtype dtype,
                    void* dst, void* stream);

/* Seeded synthetic input generator (the same counter-based SplitMix64 as synth/):
 * fills dst[r*ld + c] (r < rows, c < cols) with element (g_row0 + r, g_col0 + c) of the
 * global [*, g_cols] tensor of stream (seed, tensor_id). kind 0 = uniform in
 * [-1,1) * scale on a 24-bit grid, kind 1 = ternary {-1,0,1}; quantised RNE to dtype. */
tp_status tp_fill(void* dst, tp_dtype dtype, int64_t rows, int64_t cols, int64_t ld,
                  uint64_t seed, int tensor_id, int kind, float scale, int64_t g_row0,
                  int64_t g_col0, int64_t g_cols, void* stream);

/* out[i] = a[i] + b[i] for n elements of dtype (a Transformer block's residual connections;
 * out may alias a or b). 16-byte aligned buffers. */
tp_status tp_add(const void* a, const void* b, void* out, size_t n, tp_dtype dtype, void* stream);

/* Writes `bytes` to a scratch buffer (device) to evict L2 between timed steps. */
tp_status tp_l2_flush(void* scratch, size_t bytes, void* stream);

/* ---- instrumentation -------------------------------------------------------------------- */
/* When enabled, every GEMM launch is bracketed by CUDA events on its launching stream. */
tp_status tp_prof_enable(int on);
tp_status tp_prof_reset(void);
/* kernel_class: 0 = tcgen05 GEMM, 1 = SIMT GEMM. Synchronises the recorded events and
 * returns the summed device time (ms), the launch count and the algorithmic flops. */
tp_status tp_prof_read(int kernel_class, double* total_ms, int64_t* launches, double* flops);
/* Span trace of the recorded regions (tracing): with tp_prof_enable(1) the library
 * also records every collective of the grids' line communicators (class 2, value = elements x
 * element size) next to the GEMM launches (classes 0 / 1, value = flops), each tagged with the
 * grid rank whose call issued it. After the work completed, up to `max` spans are written to
 * out (start / end in ms relative to the earliest recorded start, in recording order); *n gets
 * the number of records. Synchronises the recorded events. */
typedef struct {
  int kernel_class;  /* 0 tcgen05 GEMM, 1 SIMT GEMM, 2 collective */
  int rank;          /* grid rank of the issuing call (-1: outside a grid call) */
  double start_ms, end_ms, value;
} tp_span;
tp_status tp_prof_spans(int max, tp_span* out, int* n);
/* Number of kernels this library has launched since load (all classes). */
int64_t tp_launch_count(void);
/* Diagnostics: when buf (device, >= 16 x uint64 per CTA of the largest grid) is non-NULL, the
 * CTA-pair GEMM writes per-CTA counters: [0] producer wait on free slots, [1] producer total,
 * [2] MMA wait on loaded stages, [3] MMA wait on a free accumulator, [4] MMA total, [5]
 * epilogue wait on accumulators, [6] epilogue total (clock64; [0],[2],[12..14] only in a
 * TP_LOOP_CLOCKS=1 build), [7]/[8]/[9] globaltimer at entry / after the prologue / at exit,
 * [10]/[11] clock64 at entry / exit. NULL disables (default). */
tp_status tp_gemm_trace(unsigned long long* buf);

/* ---- LayerNorm in the tensor-parallel layouts ------------------------ */
/* LayerNorm over the hidden (column) dimension, per row r of the global activation A [M, H]:
 *   mu = mean_c A[r,c], var = mean_c (A[r,c]-mu)^2, y = (A - mu)/sqrt(var + eps)*gamma + beta
 * (textbook definition; the paper names the layer, without a formula).
 * The activation is sharded as tensor `tensor` (TP_TENSOR_X: A = X [M, K]; TP_TENSOR_Y: A = Y
 * [M, N]) of the layer `desc` on this grid: this rank passes its dense block [rows, cols] of
 * tp_shard_extent(grid, desc, tensor) (row stride = cols). gamma / beta / dgamma / dbeta are
 * the matching column block [cols] (tp_shard_extent(..., TP_TENSOR_BIAS) for Y; the X column
 * block for X); NULL gamma = ones, NULL beta = zeros. dtype = desc->dtype.
 * Row statistics are all-reduced (fp32) over the ranks holding the other column blocks of
 * the same rows; dgamma / dbeta over the ranks holding the other row blocks of the same
 * columns. stats: [rows, 2] fp32 (mean, rstd), written by fwd, read by bwd.
 * Collective: every rank of the grid calls with identical desc / tensor / eps.
 * Errors: TP_ERR_ARG (tensor not X/Y, null pointers), TP_ERR_WORKSPACE, TP_ERR_INDIVISIBLE. */
tp_status tp_layernorm_ws_size(const tp_grid* grid, const tp_linear_desc* desc, tp_tensor tensor,
                               size_t* ws_bytes);
tp_status tp_layernorm_fwd(tp_grid* grid, const tp_linear_desc* desc, tp_tensor tensor, float eps,
                           const void* x, const void* gamma, const void* beta, void* y,
                           float* stats, void* ws, size_t ws_bytes, void* stream);
/* dx may be NULL (skip), dgamma / dbeta may be NULL (skip). */
tp_status tp_layernorm_bwd(tp_grid* grid, const tp_linear_desc* desc, tp_tensor tensor,
                           const void* dy, const void* x, const void* gamma, const float* stats,
                           void* dx, void* dgamma, void* dbeta, void* ws, size_t ws_bytes,
                           void* stream);

/* ---- Ring Self-Attention (sequence parallelism) ------------------------ */
/* softmax(Q K^T * scale) V ("Attention(Q,K,V) = softmax(QK^T/sqrt(d_k))V") for
 * `heads` independent (batch x head) problems, with Q, K, V split along the sequence over the
 * p ranks of a TP_1D grid (the ring, "the input data is split along the sequence
 * dimension"). This rank passes q, k, v and out as [heads, seq/p, d_k] row-major (rows
 * [rank*seq/p, (rank+1)*seq/p) of every head). Pass 1 circulates K blocks around the ring
 * (p-1 shifts; "transferred to the next device for N-1 times") and assembles the fp32
 * score rows, a row softmax forms the probabilities, pass 2 circulates V blocks and
 * accumulates the output. dtype TP_BF16 (tensor cores, fp32 accumulate) or
 * TP_FP32. scale 0 means 1/sqrt(d_k). Collective over the ring.
 * Errors: TP_ERR_CONSTRAINT (grid not 1D), TP_ERR_INDIVISIBLE (seq % p), TP_ERR_WORKSPACE. */
typedef struct {
  int64_t seq;    /* global sequence length s */
  int64_t d_k;    /* head dimension of Q, K and V */
  int64_t heads;  /* independent problems (batch x heads) */
  tp_dtype dtype;
  float scale;
} tp_rsa_desc;
tp_status tp_rsa_ws_size(const tp_grid* grid, const tp_rsa_desc* desc, size_t* ws_bytes);
/* lse (nullable): fp32 [heads, seq/p] - the online-softmax ring's row log-sum-exp (base 2,
 * scaled scores), written by the bf16 d_k in {64, 128} ring; with `out` it selects the fused
 * ring backward. */
tp_status tp_rsa_fwd(tp_grid* grid, const tp_rsa_desc* desc, const void* q, const void* k,
                     const void* v, void* out, float* lse, void* ws, size_t ws_bytes, void* stream);
/* Backward (the chain rule of the same definition; the paper describes the forward only):
 * given dout = dL/dout [heads, seq/p, d_k] of this rank's rows, writes dq, dk, dv (same layout).
 * With the forward's out and lse (bf16, d_k 64 / 128): the fused ring backward - K and V travel
 * the ring, each step one fused attention-backward launch (scores recomputed on chip from lse)
 * adds this rank's queries' dq (fp32) and writes the visiting block's dk / dv contributions;
 * the contributions are reduce-scattered to the blocks' owners (fp32). Otherwise the two-pass
 * form: scores recomputed with the K ring; dP uses the V ring, dq the K ring, dk / dv
 * contributions reduce-scattered. Same workspace as the forward (tp_rsa_ws_size). */
tp_status tp_rsa_bwd(tp_grid* grid, const tp_rsa_desc* desc, const void* q, const void* k,
                     const void* v, const void* out, const float* lse, const void* dout, void* dq,
                     void* dk, void* dv, void* ws, size_t ws_bytes, void* stream);

/* ---- multi-head attention core in the TP layouts ---------------------- */
/* Between a QKV linear (qkv_desc: M tokens = batch x seq, K = h, N = 3h) and the output
 * projection: per sequence and head, softmax(Q K^T scale) V (scale 0 = 1/sqrt(d)).
 * Head g occupies QKV columns [3 d g, 3 d (g+1)) as [q | k | v] (d = h / heads), so this
 * rank's QKV output block (tp_shard_extent(grid, qkv_desc, TP_TENSOR_Y), row stride = cols)
 * holds whole heads; its row extent must hold whole sequences. All work is local (no
 * communication in any mode). out: [rows, heads_local d] = the X block of the output
 * projection (1D row split, same 2D / 2.5D block, 3D parity + 1); backward takes dL/d(out)
 * in that layout and writes dL/d(qkv) in the QKV block layout. Errors: TP_ERR_SHAPE (a
 * block splits a head or a sequence, d % 8), TP_ERR_WORKSPACE. */
tp_status tp_attention_ws_size(const tp_grid* grid, const tp_linear_desc* qkv_desc, int64_t seq,
                               int64_t heads, size_t* ws_bytes);
/* lse (nullable): fp32 [heads_local x rows] (problem order: sequence-major, then head, then
 * position) - the forward's per-row log-sum-exp (base 2, scaled scores). Written by the fused
 * forward (bf16, d in {64, 128}); passing it and the forward's `out` to the backward selects the
 * fused backward (scores recomputed on chip from lse, never stored in HBM); with either NULL the
 * backward recomputes the scores two-pass through workspace. */
tp_status tp_attention_fwd(tp_grid* grid, const tp_linear_desc* qkv_desc, int64_t seq,
                           int64_t heads, float scale, const void* qkv, void* out, float* lse,
                           void* ws, size_t ws_bytes, void* stream);
tp_status tp_attention_bwd(tp_grid* grid, const tp_linear_desc* qkv_desc, int64_t seq,
                           int64_t heads, float scale, const void* qkv, const void* out,
                           const float* lse, const void* dout, void* dqkv, void* ws,
                           size_t ws_bytes, void* stream);

/* ---- analytic cost model --------------------- */
/* One linear layer, fwd+bwd, bias-free, on the grid (mode, world, q, d) with desc's M, K, N,
 * dtype, split_1d and flags (TP_FLAG_W25_DEPTH_SHARDED). Host only, no device work.
 *   paper_elems      the paper's Table tp-comm-vol row, evaluated verbatim (elements):
 *                    1D 2(p-1)S_x (S_y for the row split), 2D 3(q-1)(S_x+S_w),
 *                    2.5D 3(q-1)(S_x/d+S_w) (per plane), 3D 2(l-1)/l (S_x+S_w+S_y)
 *   counted_elems    what this library's collective schedule moves, all ranks together, in
 *                    SPEC's conventions (bcast/reduce (g-1)m, AR 2(g-1)m, AG/RS (g-1)m_total)
 *   link_bytes       per-GPU bytes over NVLink = counted_elems / world * element size
 *   flops            per-GPU flops = 6 M K N / world
 *   mem_x/w/y        per-rank at-rest elements of the X, W and Y shards
 *   t_tensor_us, t_link_us, t_roof_us   flops / peak_tflops, link_bytes / link_gbs, their max
 *   fused_direct_bytes, fused_staged_bytes   bytes one rank reads from peers per layer fwd+bwd
 *                    on the fused owner-computes path (TP_FLAG_PEER_FUSED, 2D / 2.5D replicated
 *                    W / 3D l=2; 0 elsewhere): panels TMA-read straight from the peers (each
 *                    re-read once per 256-wide output tile row / column it feeds), and staged
 *                    (TP_FLAG_PEER_STAGED: each distinct remote shard pulled once). Generic rank:
 *                    every panel remote except the rank's own shards.
 *   t_exposed_us     communication the library's schedule leaves exposed (not under a GEMM)
 *                    at those rates: per collective, received bytes / link_gbs minus the GEMM
 *                    it overlaps (0 at world == 1 or when either rate is <= 0)
 * peak_tflops / link_gbs <= 0 leave the times at 0. Errors: TP_ERR_CONSTRAINT (grid),
 * TP_ERR_INDIVISIBLE, TP_ERR_ARG (null pointers). */
typedef struct {
  double paper_elems, counted_elems, link_bytes, flops;
  double mem_x, mem_w, mem_y;
  double t_tensor_us, t_link_us, t_roof_us;
  double t_exposed_us;
  double fused_direct_bytes, fused_staged_bytes;
} tp_cost;
tp_status tp_cost_model(tp_mode mode, int world, int q, int d, const tp_linear_desc* desc,
                        double peak_tflops, double link_gbs, tp_cost* out);

#ifdef __cplusplus
}
#endif
#endif /* TP_B200_H */
