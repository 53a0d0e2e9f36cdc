// Internal structures shared by the host runtime (tq_runtime.cpp) and the
// sm_100a kernels (tq_kernels.cu).  Not part of the C-ABI.
#pragma once

#include <cstdint>
#include <cuda.h>
#include <cstdlib>
#include <utility>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

namespace tqb {

// ---- tiling constants -------------------------------------------------------
constexpr int kBM = 128;       // weight rows per tile = tcgen05 M (TMEM lanes)
constexpr int kKC = 64;        // K elements per pipeline chunk (one 128B swizzle atom of fp16)
constexpr int kBNMax = 192;    // tokens per tile (tcgen05 N, multiple of 16, <= 256)
constexpr int kDenseBits = 16; // "bits" value of a dense fp16 weight (projection pass)

// Bytes of one (weight, m-block, k-chunk) code block: 128 rows x 64 codes.
__host__ __device__ constexpr int code_block_bytes(int bits) { return kBM * kKC * bits / 8; }

// One work unit of the grouped tcgen05 GEMM: a 128-row m-block of one weight
// matrix against up to kBNMax activation rows, over a K-chunk range.
struct alignas(16) Unit {   // 16-byte aligned: written / read as two 128-bit words
    int32_t weight;    // weight matrix index (routed e, K+s for shared s, 0 for projection)
    int32_t mb;        // m-block (rows mb*128 ..)
    int32_t x_row;     // first activation row (X / Ext matrices)
    int32_t n_tok;     // valid activation rows (1..kBNMax)
    int32_t y_row;     // first output row in the split buffer
    int16_t kc_begin;  // main K chunks [kc_begin, kc_end)
    int16_t kc_end;
    int16_t n_ext;     // extension chunks appended after the main chunks
    int16_t split;     // split-K index (selects the output buffer)
    int32_t pad;
};
static_assert(sizeof(Unit) == 32, "Unit is 32 bytes");

// Parameters of one launch of the grouped GEMM (passed as __grid_constant__).
struct GemmParams {
    CUtensorMap tmap_x64;   // activations fp16 [rows, k_pad], box 64 rows x 64 cols, SW128
    CUtensorMap tmap_e64;   // extension activations fp16 [rows, ext_cols], box 64 x 64
    CUtensorMap tmap_x16;   // the same tensors with 16-row boxes (small token tiles)
    CUtensorMap tmap_e16;
    const __half* x_ptr;    // the same two matrices for the cp.async path (small token tiles)
    int64_t x_ld;
    const __half* e_ptr;
    int64_t e_ld;
    int32_t contig;         // 1: each CTA takes a contiguous unit range (runs share activation tiles)
    int32_t e_slots;        // extension-block ring depth (1 or 2)
    int32_t xr_slots;       // resident activation slots (decode config): max chunks per unit
    int64_t x_atom_rows;    // > 0: x_ptr / e_ptr are atom-major [cols/64][x_atom_rows][64 halves], rows
                            // pre-swizzled (128B pattern of the row index), tile rows 8-aligned:
                            // activation tiles are plain bulk copies, one per 64-column atom
    const uint8_t* codes;   // [weight][mb][kc] blocks of code_block_bytes(bits)
    int64_t weight_stride;  // bytes per weight matrix in `codes`
    const __half* scales;   // [weight][mb][G][128] fp16 scale slabs (quantized weights)
    const uint8_t* ext_blocks;  // [weight][mb][n_ext64] dense fp16 extension blocks (-zero*s | U_p codes)
    int32_t n_ext64;            // extension blocks per (weight, m-block) (0: none)
    const float* w_outscale;    // per weight: epilogue multiplier (2^-k)
    const Unit* units;
    const int32_t* n_units;     // device counter (units are built on the device)
    float* y;                   // output, split buffers of y_split_stride floats
    int64_t y_split_stride;
    int32_t ldy;                // output row stride (floats)
    int32_t o_valid;            // valid weight rows (outputs written only below)
    int32_t o_pad;
    int32_t bits;               // 2,3,4,8 or 16 (dense fp16)
    int32_t group_size;
    int32_t groups;             // G
    int32_t rank;               // r
    int32_t kc_total;
    int32_t kc_width;           // K elements per pipeline chunk: 64 or 128
    int32_t dn;                 // TMEM accumulator columns per buffer (64, 128 or 192)
    int32_t n_ext_chunks;       // extension chunks of units that carry them
    int32_t bn_max;             // largest token tile of the launch (sizes the activation ring)
    int32_t x_stage_rows;       // set by launch_gemm
    int32_t x_stages;           // set by launch_gemm
    int32_t c_stages;           // set by launch_gemm
    int32_t group_shift;        // log2(group_size) or -1, set by launch_gemm
    int32_t debug;              // TQ_DEBUG bits (profiling only): 1 no dequant, 2 no MMA, 4 no stores, 8 trace
    unsigned long long* trace;  // trace buffer (TQ_DEBUG & 8)
};

// ---- kernel argument blocks -------------------------------------------------
struct PlanArgs {
    const int32_t* ids;
    int batch, top_k, num_experts;
    int e_begin, e_end;        // resident routed experts
    int num_shared;            // shared experts (weights K..K+S-1), rows after the slots
    int mb_count;              // m-blocks of the expert weights
    int kc_total, nsplit, n_ext;   // nsplit: upper bound; the kernel picks the best <= nsplit
    int nsplit_min;            // lower bound (resident activation tiles must fit shared memory)
    float split_cost;          // extra output traffic of one more split, relative to the weight bytes
    int run_order;             // 1: units ordered (expert, tile, split, m-block): runs of m-blocks
    int proj_bn;               // token tile of the projection pass (0: bn)
    int ext8;                  // the ext chunk's cost in 1/8 main chunks: K splits balanced with it (0: uniform)
    int max_run;               // > 0: most chunks (main + ext) one unit may carry (resident activation slots)
    int unit_cost8;            // > 0: choose the K split by per-CTA time with a per-unit cost of unit_cost8/8 chunks
    int main_kc;               // 1: main chunks present (0 for the lotile-only path)
    int num_sms;               // persistent grid size (load-balance target)
    int bn;                    // token tile (<= kBNMax)
    int32_t* nsplit_out;       // chosen split count (read by combine), may be null
    int proj_mb, proj_kc_total, proj_nsplit;  // projection pass (0 mb -> none)
    int32_t* perm;
    int32_t* inv;
    int32_t* offsets;
    int32_t* poffsets;         // K+1: expert row bases in the 8-row padded activation layout
    Unit* units;
    int32_t* n_units;
    Unit* proj_units;
    int32_t* n_proj_units;
    int32_t* err_flag;
};

struct GatherArgs {
    const __half* x16;       // [B][k_pad]
    const float* sx;         // [B][G]
    const float* zpart;      // [proj_nsplit][B][zcols]
    int64_t zsplit_stride;
    int zcols, proj_nsplit;
    const int32_t* ids;
    const int32_t* perm;
    const int32_t* offsets;  // K+1 (offsets[K] = slots)
    const int32_t* pm_of;    // per routed expert: projection matrix index
    const float* zscale;     // per routed expert: su_p * inv_scalar * 2^k_e
    const float* rowscale;   // per projection row: 2^k normalisation
    int batch, top_k, num_experts, k_pad, groups, rank, ext_cols;
    int with_shared;         // append B shared-expert rows
    int use_sx, use_z;       // path selection
    __half* xp;              // [rows][k_pad], or atom-major (see atom_rows)
    __half* ep;              // [rows][ext_cols], or atom-major
    const int32_t* poffsets; // if set: slot s of expert e goes to padded row s + poffsets[e] - offsets[e]
    int64_t atom_rows;       // > 0: atom-major, 128B-swizzled layout [cols/64][atom_rows][64] (bulk-copy tiles)
    const int32_t* inv;      // token-major gather: slot of flat routing index f (-1: invalid id)
};

// dequant_only comparison layout (tq_layouts.cu)
struct DequantAllArgs {
    const uint8_t* codes;      // repacked code blocks [w][mb][kb64]
    int64_t weight_stride;     // bytes per weight
    const uint16_t* scales;    // [w][mb][G][128] prescaled fp16
    const uint8_t* ext_blocks; // [w][mb] n_ext64 dense blocks; columns [0, G) = -zero * s'
    int64_t ext_bytes;         // bytes per (w, mb)
    const float* w_outscale;   // 2^-k per weight
    __half* out;               // [w][o][i] fp16
    int64_t o, i;
    int n_weights, mb_count, kb_total, groups, group_size;
};

struct CombineArgs {
    const float* y;          // split buffers [nsplit][rows][o]
    int64_t split_stride;
    int nsplit;
    const int32_t* inv;
    const float* gates;
    const int32_t* offsets;  // K+1
    const int32_t* ids;      // with poffsets: routed row = inv + poffsets[e] - offsets[e]
    const int32_t* poffsets;
    int num_experts, batch, top_k, out_dim, num_shared;
    int use_routed;
    const float* ysh;        // shared-expert rows: split buffers, row = sh_row0 + s*batch + b
    int64_t sh_split_stride;
    int sh_nsplit;
    int sh_from_offsets;     // 1: sh_row0 = offsets[num_experts] (single-GPU layout), 0: 0
    const int32_t* nsplit_dev;  // if set: split count of both routed and shared rows (chosen by plan)
    float* out;
};

// ---- decode path (tq_decode.cu): route+scatter -> fused expert GEMM -> combine ----
//
// Slot layout: routed expert e owns activation rows [e * cap8, e * cap8 + cnt[e]),
// shared expert s the rows [(K + s) * cap8, ... + batch) (row b = token b).  The
// rows live in the atom-major, 128B-pre-swizzled layout [k/64][atom_rows][64]
// (one bulk copy per 64-column atom lands a token tile MMA-ready).
constexpr int kDecMaxW = 128;        // routed + shared weights
constexpr int kDecMaxTopK = 8;       // destinations per token held in shared memory

struct DecRouteArgs {
    const float* x;                  // [B][i] f32
    int batch, in_dim, k_pad;
    const float* gate;               // [K][i] router
    int num_experts, top_k, num_shared;
    int given;                       // 1: routing given (ids_in / gates_in), no scoring
    const int32_t* ids_in;
    int32_t* ids;                    // computed routing (given == 0)
    float* gates;
    float* score_ws;                 // [B][K]
    int32_t* ticket;                 // [B] per-token CTA tickets (self-resetting)
    int group_size, groups, rank, num_q;
    const int8_t* vcodes;            // [N][r][i] tiled.v.codes
    const float* vscale;             // [N][r] sigma_j * (vabs_q / 127)
    const int32_t* q_tier;           // [N] 0 folded, 1 scalar, 2 general, -1 unused
    const int32_t* q_first;          // [N] expert whose scaling defines the folded s_q
    const float* scaling;            // [K][i]
    const int32_t* e_q;              // [K] tile column q(e)
    const float* zscale;             // [K] su_p * inv_scalar * 2^k_e
    float* zq_ws;                    // [B][N][r] projections of the folded / scalar column blocks
    int use_main, use_lr;            // path: residual (group sums) / low-rank (projections)
    int cap8;                        // rows per weight in the slot layout
    int64_t atom_rows;
    int ext_cols;                    // ext row width (multiple of 64)
    __half* xperm;                   // slot rows, atom-major [k_pad/64][atom_rows][64]
    __half* extperm;                 // ext rows [Sx | Z * zscale | 0], atom-major [ext_cols/64][atom_rows][64]
    int32_t* cnt;                    // [K] slots taken per routed expert (zeroed by the combine)
    int32_t* inv;                    // [B * top_k] slot row of (b, t), -1 for an invalid id
    int32_t* err_flag;
    unsigned long long* trace;       // TQ_ROUTE_TRACE builds only: [cta][16] globaltimer
};

struct DecParams {
    const uint8_t* codes;            // [w][mb][kb64] code blocks
    int64_t weight_stride;
    const __half* scales;            // [w][mb][G][128]
    const uint8_t* ext_blocks;       // [w][mb][E64] dense fp16 128 x 64 blocks [-zero*s' | U_p | 0]
    int n_ext64;
    const float* w_outscale;         // [w] 2^-k
    int bits, group_size, groups, group_shift;
    int kc64;                        // k_pad / 64
    int nmain;                       // main steps (256 K each) per segment; 0 = low-rank only path
    int mb_count, o_valid;
    int num_experts, num_shared, batch;
    const int32_t* cnt;
    int cap8;
    int64_t atom_rows;
    const __half* xperm;
    const __half* extperm;
    float* yslot;                    // [(K + S) * cap8][o] expert rows
    int ldy;
    float* scratch;                  // [grid][2][dn][128] split-segment partials
    int32_t* seg_cnt;                // per segment arrivals (self-resetting)
    int code_stages, x_stages, code_stage_bytes;   // set by launch_decode
    unsigned long long* trace;       // TQ_DEC_TRACE builds only
    int trace_cta;
    int check_slots;                 // TQ_DEC_CHECK builds: expected routed slots (batch * top_k)
};

struct DecCombineArgs {
    const float* yslot;
    int ldy;
    const int32_t* inv;
    const float* gates;
    int batch, top_k, out_dim, num_shared, num_experts, cap8;
    int32_t* cnt;                    // zeroed here for the next forward
    float* out;
};

// ---- host-side tables the runtime keeps for a loaded layer ----------------------
struct DeviceBuf {
    void* ptr = nullptr;
    size_t bytes = 0;
};

// kernel launch through cudaLaunchKernelEx (no launch attributes: programmatic
// dependent launch was measured and gave nothing on this path)
template <typename... KArgs, typename... Args>
inline cudaError_t launch_maybe_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                                    Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cfg.attrs = nullptr;
    cfg.numAttrs = 0;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

}  // namespace tqb
