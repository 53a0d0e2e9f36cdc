/*
 * tileq_b200.h -- C-ABI of the B200-native fused low-rank MoE inference
 * engine (libtileq_b200.so).  Plain pointers and sizes only; no C++ or
 * torch types cross this boundary and no exception escapes it.
 *
 * Every entry point names the reference interface it replaces
 * (paths relative to /root/reference/proj):
 *
 *   tq_layer_load      <- read_artifact(dir, verify_crc)        include/tileq/io.hpp:55,  src/io.cpp:679-813
 *   tq_layer_create    <- an in-memory TileQLayer               include/tileq/infer.hpp:22-28 (QuantizedExpert
 *                         quant.hpp:37-63, TiledLowRank tiler.hpp:45-56, CodedBlock codec.hpp:42-50)
 *   tq_artifact_check  <- read_artifact's validation alone (no device), src/io.cpp:186-295,422-485,679-813
 *   tq_route           <- route(x, gate_weights, top_k)         include/tileq/moe.hpp:53, src/moe.cpp:43-89
 *   tq_permute         <- (no counterpart: the per-token loop of reference_forward, src/moe.cpp:106-133)
 *   tq_forward         <- tileq_forward / qmoe_forward / lotile_forward
 *                                                               include/tileq/infer.hpp:52-73, src/infer.cpp:40-185
 *   tq_forward_routed  <- forward_from_artifact's route + tileq_forward
 *                                                               bindings/py_module.cpp:112-117
 *   tq_unpack_codes    <- unpack_codes(bytes, bits, count)      include/tileq/codec.hpp:68, src/codec.cpp:168-195
 *   tq_launch_count    <- dispatch_count()                      include/tileq/infer.hpp:37-38 (GPU analogue:
 *                                                               kernel launches per forward, constant in B)
 *   tq_layout_forward  <- bench()'s layouts: lotile_forward / baseline_1d_forward /
 *                         baseline_elementwise_forward / dequantize-all
 *                                                               include/tileq/infer.hpp:77-131, src/infer.cpp:187-426
 *   tq_dequantize_experts <- dequantize(residual) for every resident expert
 *                                                               include/tileq/quant.hpp, src/quant.cpp:285-323
 *
 * Status codes mirror the reference error taxonomy (include/tileq/errors.hpp:13-50)
 * with the same triggering conditions; the message (tq_last_error, thread
 * local) names the offending tensor or field like the reference's what().
 *
 * Pointers marked [dev] are CUDA device pointers on the layer's device;
 * [host] are host pointers.  `stream` is a cudaStream_t (NULL = legacy
 * default stream).  All device entry points are asynchronous and
 * stream-ordered; a layer may be used from one stream at a time.
 */
#ifndef TILEQ_B200_H
#define TILEQ_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    TQ_OK = 0,
    TQ_ERR_SHAPE = 1,    /* ShapeError   */
    TQ_ERR_PARAM = 2,    /* ParamError   */
    TQ_ERR_SIZE = 3,     /* SizeError    */
    TQ_ERR_FORMAT = 4,   /* FormatError  */
    TQ_ERR_IO = 5,       /* IoError      */
    TQ_ERR_NUMERIC = 6,  /* NumericError */
    TQ_ERR_DATA = 7,     /* DataError    */
    TQ_ERR_CUDA = 8,     /* CUDA runtime / launch failure       */
    TQ_ERR_NCCL = 9,     /* collective failure (expert parallel) */
    TQ_ERR_INTERNAL = 99
} tq_status;

typedef enum {
    TQ_PATH_FULL = 0,    /* tileq_forward  = qmoe + lotile (infer.cpp:182-185) */
    TQ_PATH_QMOE = 1,    /* qmoe_forward   (infer.cpp:40-51)                   */
    TQ_PATH_LOTILE = 2   /* lotile_forward (infer.cpp:53-180)                  */
} tq_path;

typedef struct tq_layer tq_layer;

typedef struct {
    int64_t num_experts;   /* K  (MoELayerSpec, moe.hpp:16-25) */
    int64_t top_k;
    int64_t in_dim;        /* i */
    int64_t out_dim;       /* o */
    int64_t num_shared;    /* S */
    int64_t rank;          /* r  (TiledLowRank::rank)          */
    int64_t grid_rows;     /* M */
    int64_t grid_cols;     /* N */
    int64_t bits;          /* residual code width              */
    int64_t group_size;    /* g */
    int64_t expert_begin;  /* resident routed experts [begin, end) (expert parallel) */
    int64_t expert_end;
    int64_t device;
    int64_t device_bytes;  /* HBM held by the layer (weights + tables) */
    int64_t tier_folded;   /* column blocks per descale tier (infer.cpp:74-99) */
    int64_t tier_scalar;
    int64_t tier_general;
} tq_layer_info;

/* Thread-local message of the last failing call on this thread. */
const char* tq_last_error(void);

/* Library build string (arch, git hash if known). */
const char* tq_version(void);

/* Load an artifact directory written by the reference's write_artifact
 * (io.cpp:565-677) onto `device`, validating it exactly like read_artifact
 * (manifest version/kind, per-tensor dtype/shape/byte_length, CRC32 unless
 * verify_crc == 0, placement bounds/injectivity/L1, positive scales, clean
 * padding bits), then repacking the residual codes, scales, zero points and
 * factor blocks into the engine's TMA tile layout in HBM.
 * expert_begin/expert_end select the resident routed experts (expert
 * parallel); pass 0, -1 for all.  Router, factors, scaling and shared
 * experts are always resident. */
tq_status tq_layer_load(const char* dir, int device, int verify_crc, int64_t expert_begin,
                        int64_t expert_end, tq_layer** out);

/* Validate an artifact directory exactly like tq_layer_load (same status
 * codes and messages) without touching any device: the host half of
 * read_artifact.  Lets a CPU-only process vet artifacts. */
tq_status tq_artifact_check(const char* dir, int verify_crc);

typedef enum { TQ_QUANT_SCALAR = 0, TQ_QUANT_VECTOR = 1 } tq_quant_mode;   /* QuantMode, quant.hpp:30 */

/* One residual matrix (QuantizedExpert, quant.hpp:37-63), host memory. */
typedef struct {
    int64_t out_dim, in_dim;      /* o x i */
    int bits;                     /* 2, 3, 4, 8 */
    int mode;                     /* tq_quant_mode */
    const uint8_t* packed;        /* LSB-first code stream (codec.cpp:150-195) */
    int64_t packed_bytes;
    /* scalar mode: o x ceil(i/g) grids, row-major */
    int64_t group_size;
    const uint16_t* scale_bits;   /* binary16 patterns of QuantGrid::scale */
    const uint8_t* zeros;         /* QuantGrid::zero_point, in [0, 2^bits) */
    /* vector mode */
    int64_t sub_dim;
    const uint16_t* codebook_bits;   /* 2^bits x sub_dim binary16 patterns */
} tq_qmat_desc;

/* An in-memory TileQLayer (infer.hpp:22-28), host memory; nothing is
 * retained after tq_layer_create returns. */
typedef struct {
    int64_t num_experts, top_k, in_dim, out_dim, num_shared;   /* MoELayerSpec */
    const float* gate_weights;       /* K x i */
    int64_t grid_rows, grid_cols, rank;                        /* M, N, r */
    const uint32_t* placement;       /* K x 2: assignment.placed[k] = (p, q) */
    const float* scaling;            /* K x i: scaling.s[k] */
    const uint16_t* singular_bits;   /* r binary16 patterns */
    const int8_t* u_codes;           /* M blocks, each o x r row-major */
    const float* u_absmax;           /* M */
    const int8_t* v_codes;           /* N blocks, each r x i row-major */
    const float* v_absmax;           /* N */
    const tq_qmat_desc* experts;     /* K routed residuals */
    const tq_qmat_desc* shared;      /* num_shared shared experts */
} tq_layer_desc;

/* Build a device-resident layer from an in-memory TileQLayer (the C++ shim's
 * entry: tileq_forward(x, layer, routing) on a layer that never touched disk).
 * Validation mirrors what the reference enforces on the same fields:
 * out-of-grid cells -> TQ_ERR_FORMAT (infer.cpp:65-72), non-positive scales
 * -> TQ_ERR_FORMAT, bits outside {2,3,4,8} -> TQ_ERR_PARAM (quant.cpp:18-22),
 * mismatched residual dims -> TQ_ERR_SHAPE. */
tq_status tq_layer_create(const tq_layer_desc* desc, int device, int64_t expert_begin, int64_t expert_end,
                          tq_layer** out);
tq_status tq_layer_free(tq_layer* layer);
tq_status tq_layer_info_get(const tq_layer* layer, tq_layer_info* out);

/* Pre-size the batch workspace for up to max_tokens tokens so the forward
 * path performs no allocation. */
tq_status tq_layer_reserve(tq_layer* layer, int64_t max_tokens);

/* route(): ids [dev] int32 batch x top_k (row-major b*top_k+t), gates [dev]
 * f32 batch x top_k.  x [dev] f32 batch x in_dim.  Bit-exact ids; gates
 * within 1 f32 ulp of the reference (moe.cpp:64-87). */
tq_status tq_route(tq_layer* layer, const float* x, int64_t batch, int32_t* ids, float* gates,
                   void* stream);

/* route() on raw arrays without a layer (the reference's standalone
 * route(x, gate_weights, top_k), moe.hpp:53): x [dev] f32 batch x in_dim,
 * gate [dev] f32 num_experts x in_dim.  top_k outside [1, num_experts] ->
 * TQ_ERR_PARAM. */
tq_status tq_route_raw(const float* x, int64_t batch, int64_t in_dim, const float* gate, int64_t num_experts,
                       int64_t top_k, int32_t* ids, float* gates, void* stream);

/* tq_route_raw on HOST arrays (the reference's route() signature in plain
 * memory, moe.hpp:53): ids [host] int64 batch x top_k, gates [host] f32.
 * Synchronous; allocates its own device staging (not a hot-path entry). */
tq_status tq_route_host(const float* x, int64_t batch, int64_t in_dim, const float* gate, int64_t num_experts,
                        int64_t top_k, int device, int64_t* ids, float* gates);

/* Stable token permutation by expert: perm [dev]
 * int32 batch*top_k (perm[pos] = b*top_k+t), offsets [dev] int32 K+1,
 * inv [dev] int32 batch*top_k (inv[f] = pos).  ids [dev] int32. */
tq_status tq_permute(tq_layer* layer, const int32_t* ids, int64_t batch, int32_t* perm,
                     int32_t* offsets, int32_t* inv, void* stream);

/* Forward with a given routing: y [dev] f32 batch x out_dim.
 * x [dev] f32, ids [dev] int32, gates [dev] f32.  Expert ids outside
 * [0, K) make the call fail with TQ_ERR_PARAM (reference_forward,
 * moe.cpp:111-114) -- checked on the device, reported on the next sync
 * point (tq_sync). */
tq_status tq_forward(tq_layer* layer, const float* x, int64_t batch, const int32_t* ids,
                     const float* gates, float* y, int path, void* stream);

/* route + forward: the reference Python binding's forward_from_artifact
 * path (py_module.cpp:112-117) on device buffers.  ids/gates may be NULL. */
tq_status tq_forward_routed(tq_layer* layer, const float* x, int64_t batch, float* y,
                            int32_t* ids, float* gates, int path, void* stream);

/* Same with HOST buffers: copies in, runs, copies out, synchronizes.
 * x [host] f32, y [host] f32, ids [host] int64 (reference dtype), gates
 * [host] f32 (ids/gates may be NULL). */
tq_status tq_forward_host(tq_layer* layer, const float* x, int64_t batch, float* y,
                          int64_t* ids, float* gates, int path);

/* tileq_forward / qmoe_forward / lotile_forward (infer.hpp:52-73) on HOST
 * buffers with a caller-supplied routing (RoutingDecision, moe.hpp:39-47):
 * x [host] f32 batch x in_dim, ids [host] int64 batch x top_k (the
 * reference's size_t expert_ids), gates [host] f32 batch x top_k, y [host]
 * f32 batch x out_dim.  An id outside [0, K) -> TQ_ERR_PARAM with
 * reference_forward's message (moe.cpp:111-114).  Synchronous. */
tq_status tq_forward_host_ids(tq_layer* layer, const float* x, int64_t batch, const int64_t* ids,
                              const float* gates, float* y, int path);

/* Waits for `stream` and reports any device-side error flag raised by the
 * layer's kernels since the last sync (e.g. expert id out of range). */
tq_status tq_sync(tq_layer* layer, void* stream);

/* Diagnostics: copy the decode path's self-resetting device counters to the host
 * (slot counts [K], router tickets [reserved batch], split-segment arrivals
 * [(K + S) * m-blocks]); every entry reads zero between forwards. */
tq_status tq_debug_decode_counters(tq_layer* layer, int32_t* out, int64_t n);

/* Test hook: the routers' f64 exp (the softmax of route(), moe.cpp:72 std::exp,
 * glibc's algorithm restated in csrc/tq_exp.h) on x [dev] f64 n -> y [dev] f64,
 * for the exp-vs-glibc parity test. */
tq_status tq_exp_f64(const double* x, int64_t n, double* y, void* stream);

/* GPU unpack of a packed stream (codec.cpp:168-195): bytes [dev], out [dev]
 * uint32 count.  Returns TQ_ERR_PARAM on a bad width or byte count and
 * TQ_ERR_FORMAT on nonzero padding bits (after synchronizing). */
tq_status tq_unpack_codes(const uint8_t* bytes, int64_t nbytes, int bits, int64_t count,
                          uint32_t* out, void* stream);

/* Decode the engine's repacked tile layout of routed expert e (or shared
 * expert e-K) back into row-major uint32 codes [dev] o x i, to prove the
 * loader's repack is bit-exact with unpack_codes. */
tq_status tq_layer_export_codes(tq_layer* layer, int64_t e, uint32_t* out, void* stream);

/* Device-time instrumentation of the fused expert GEMM (the dominant
 * kernel): when enabled, every expert-GEMM launch is bracketed by CUDA events
 * on its launching stream; tq_gemm_time_get returns the accumulated device
 * milliseconds and launch count since the last enable (synchronizes). */
tq_status tq_gemm_timing_enable(tq_layer* layer, int enable);
tq_status tq_gemm_time_get(tq_layer* layer, double* ms_total, int64_t* launches);

/* Kernel launches issued by this layer since the last reset (GPU analogue
 * of dispatch_count(), infer.hpp:37-38). */
uint64_t tq_launch_count(const tq_layer* layer);
void tq_reset_launch_count(tq_layer* layer);

/* ---- comparison layouts (the paper's bench, infer.cpp:345-426) --------- */

/* The bench layouts (BenchLayout, infer.hpp:113). */
typedef enum {
    TQ_LAYOUT_FUSED_2D = 0,     /* lotile_forward: the engine's fused low-rank path        */
    TQ_LAYOUT_SHARED_1D = 1,    /* baseline_1d_forward on shared_1d_from_tiled_representative */
    TQ_LAYOUT_ELEMENT_WISE = 2, /* baseline_elementwise_forward on elementwise_factors_from_tiled */
    TQ_LAYOUT_DEQUANT_ONLY = 3  /* dequantize() every resident routed expert                 */
} tq_layout;

/* Prepare a layout's factors / buffers once, outside any timed region, as
 * bench() does (infer.cpp:381-387).  tq_layout_forward prepares on first use. */
tq_status tq_layout_prepare(tq_layer* layer, int layout);

/* One call of a layout on a GIVEN routing: x [dev] f32 batch x in_dim, ids
 * [dev] int32 / gates [dev] f32 batch x top_k, y [dev] f32 batch x out_dim
 * (ignored by DEQUANT_ONLY).  *dispatches [host, may be NULL] receives the
 * reference-style dispatch count of the call (matrix multiplies:
 * fused 2, 1D 1 + B*top_k, element-wise 2*B*top_k, dequant 0; the kernel
 * launches are in tq_launch_count). */
tq_status tq_layout_forward(tq_layer* layer, int layout, const float* x, int64_t batch, const int32_t* ids,
                            const float* gates, float* y, int64_t* dispatches, void* stream);

/* Every resident routed expert's residual, dequantized: out [dev] fp16
 * [n_experts][out_dim][in_dim] (the DEQUANT_ONLY layout's work). */
tq_status tq_dequantize_experts(tq_layer* layer, uint16_t* out, void* stream);

/* ---- expert-parallel stages (EP host orchestration in Python calls these
 * around its NCCL all-to-all exchange) ------------- */

/* Build the dispatch rows for locally routed tokens: per permuted slot
 * pos, row pos of xrows [dev] fp16 (batch*top_k x in_pad) and of extrows
 * [dev] fp16 (batch*top_k x ext) -- token activations plus the rank-r
 * projection and group sums the owning rank needs (computed here, since
 * the factor blocks are replicated). */
tq_status tq_ep_dispatch_rows(tq_layer* layer, const float* x, int64_t batch,
                              const int32_t* ids, const int32_t* perm, uint16_t* xrows,
                              uint16_t* extrows, int path, void* stream);

/* Expert compute on received rows: segments [host] int64 triplets
 * (local_expert, row_begin, row_count) sorted by row_begin; yrows [dev] f32
 * (rows x out_dim). */
tq_status tq_ep_expert_rows(tq_layer* layer, const uint16_t* xrows, const uint16_t* extrows,
                            int64_t rows, const int64_t* segments, int64_t nseg, float* yrows,
                            int path, void* stream);

/* Combine returned rows (in permuted-slot order) with the gates plus the
 * shared experts applied to the home tokens: y [dev] f32 batch x out_dim. */
/* Expert outputs for rows received in FIXED-CAPACITY slabs (decode-sized expert
 * parallel, equal-split all-to-alls, no host round trip): rows [dev] fp16
 * [n_src * slab][row_ld], each row [x (tq_ep_xrow_elems) | ext (tq_ep_extrow_elems)];
 * source s's rows for local expert j start at s * slab + sum_{j' < j} counts[s][j'];
 * counts [dev] int32 [n_src][e_stride] (the received count matrix).  Work units are
 * built on the device from counts; yrows [dev] f32 [n_src * slab][out_dim] (rows past
 * a source's count are not written).  Stream-ordered, no synchronization. */
tq_status tq_ep_expert_rows_slab(tq_layer* layer, const uint16_t* rows, int64_t row_ld, int64_t n_src, int64_t slab,
                                 const int32_t* counts, int64_t e_stride, float* yrows, int path, void* stream);

tq_status tq_ep_combine(tq_layer* layer, const float* x, int64_t batch, const float* yrows,
                        const int32_t* inv, const float* gates, float* y, int path,
                        void* stream);

/* Row widths of the dispatch buffers (fp16 elements). */
int64_t tq_ep_xrow_elems(const tq_layer* layer);
int64_t tq_ep_extrow_elems(const tq_layer* layer);

/* ------------------------------------------------------------------------
 * Artifact producer hot spots, device arrays, bit-identical to
 * the reference.  Quantized experts cross as unpacked codes (uint8, rows x
 * cols), per-group scales (f32, binary16-exact) and zero points (int32),
 * rows x ceil(cols / group_size), row-major.  These calls synchronize the
 * stream where the reference returns a host value or may throw.
 *
 *   tq_estimate_hessian <- estimate_hessian(calib, damping_fraction)
 *                          include/tileq/quant.hpp:67, src/quant.cpp:116-150
 *   tq_spd_inverse      <- spd_inverse(h) (internal)   src/quant.cpp:72-112
 *   tq_quantize_rtn     <- quantize_rtn(r, bits, group_size)
 *                          include/tileq/quant.hpp:74, src/quant.cpp:152-175
 *   tq_quantize_gptq    <- quantize_gptq(r, h, bits, group_size)
 *                          include/tileq/quant.hpp:85-86, src/quant.cpp:177-221
 *   tq_proxy_loss       <- proxy_loss(original, q, h)
 *                          include/tileq/quant.hpp:104, src/quant.cpp:325-343
 *   tq_sketch_lowrank   <- sketch_lowrank(w, rank, power_iters, seed)
 *                          include/tileq/lowrank.hpp:21-30, src/lowrank.cpp:194-247
 *                          (extract_features tiler.cpp:137, decompose_shared tiler.cpp:308)
 * ------------------------------------------------------------------------ */

/* calib [dev] f32 tokens x dim -> h [dev] f32 dim x dim; *damping_out (host,
 * nullable) = lambda.  Empty set -> TQ_ERR_DATA; damping < 0 -> TQ_ERR_PARAM. */
tq_status tq_estimate_hessian(const float* calib, int64_t tokens, int64_t dim, double damping_fraction, float* h,
                              double* damping_out, void* stream);

/* h [dev] f32 n x n -> hinv [dev] f64 n x n.  A non-positive or non-finite
 * pivot -> TQ_ERR_NUMERIC with the reference's message. */
tq_status tq_spd_inverse(const float* h, int64_t n, double* hinv, void* stream);

/* r [dev] f32 rows x cols -> codes / scales / zeros [dev]. */
tq_status tq_quantize_rtn(const float* r, int64_t rows, int64_t cols, int bits, int64_t group_size, uint8_t* codes,
                          float* scales, int32_t* zeros, void* stream);

/* r [dev] f32 rows x cols, h [dev] f32 cols x cols -> codes / scales / zeros
 * [dev]; *used_rtn (host, nullable) = 1 when plain rounding won the proxy-loss
 * comparison (quant.cpp:216-219).  One working row and its grids must fit in
 * shared memory (cols up to ~27000). */
tq_status tq_quantize_gptq(const float* r, int64_t rows, int64_t cols, const float* h, int bits, int64_t group_size,
                           uint8_t* codes, float* scales, int32_t* zeros, int32_t* used_rtn, void* stream);

/* sketch_lowrank(w, rank, power_iters, seed) (include/tileq/lowrank.hpp:21-30,
 * src/lowrank.cpp:194-247): w [dev] f32 rows x cols -> left [dev] f32 rows x rank,
 * right [dev] f32 rank x cols, singulars [dev] f32 rank (nonincreasing).  The f64
 * working copy stays on the device (8 * rows * cols bytes); the probes are drawn
 * on the host with the reference's generator.  Synchronizes the stream. */
tq_status tq_sketch_lowrank(const float* w, int64_t rows, int64_t cols, int64_t rank, int power_iters, uint64_t seed,
                            float* left, float* right, float* singulars, void* stream);

/* tr(E H E^T), E = original - dequantize(codes, scales, zeros), into *loss (host). */
tq_status tq_proxy_loss(const float* original, int64_t rows, int64_t cols, const uint8_t* codes, const float* scales,
                        const int32_t* zeros, int bits, int64_t group_size, const float* h, double* loss,
                        void* stream);

#ifdef __cplusplus
}
#endif
#endif /* TILEQ_B200_H */
