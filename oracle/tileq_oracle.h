/* TEST INFRASTRUCTURE ONLY -- the checker, never the product.
 *
 * Plain-C restatement of the reference's fused low-rank MoE inference path
 * (/root/reference/proj).  Every function cites the reference lines it
 * follows and reproduces its arithmetic (f64 accumulation order, rounding
 * points) so that results are bit-identical to the compiled reference; this
 * is checked in tests/test_oracle.py against oracle/_ref/libtileq_ref.so and
 * against the frozen values of the reference's own tests (tests/golden/).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library.
 */
#ifndef TILEQ_ORACLE_H
#define TILEQ_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes mirror the reference error taxonomy (errors.hpp:13-50) */
enum { TQO_OK = 0, TQO_SHAPE = 1, TQO_PARAM = 2, TQO_FORMAT = 4 };

float tqo_half_to_float(uint16_t bits);
uint16_t tqo_float_to_half(float value);
int64_t tqo_packed_byte_length(int64_t count, int bits);
int tqo_unpack_codes(const uint8_t* bytes, int64_t nbytes, int bits, int64_t count, uint32_t* out);
int tqo_pack_codes(const uint32_t* codes, int64_t count, int bits, uint8_t* out);
uint32_t tqo_crc32(const uint8_t* data, int64_t n);

/* One scalar-mode quantized matrix as stored on the wire (quant.hpp:37-63). */
typedef struct {
    const uint8_t* packed;    /* o*i codes, LSB-first, `bits` each          */
    const uint16_t* scales;   /* o * groups binary16 patterns               */
    const uint32_t* zeros;    /* o * groups unpacked zero points            */
    int bits;
    int64_t group_size;
} tqo_qmat;

int tqo_dequantize_rows(const tqo_qmat* q, int64_t out_dim, int64_t in_dim, int64_t r0,
                        int64_t r1, float* out);

int tqo_route(const float* x, int64_t batch, int64_t in_dim, const float* gate,
              int64_t num_experts, int64_t top_k, int64_t* ids, float* gates);

int tqo_permute(const int64_t* ids, int64_t batch, int64_t top_k, int64_t num_experts,
                int32_t* perm, int32_t* offsets, int32_t* inv);

int tqo_qmoe_forward(const float* x, int64_t batch, int64_t in_dim, int64_t out_dim,
                     int64_t num_experts, int64_t num_shared, int64_t top_k,
                     const tqo_qmat* experts /* K + S */, const int64_t* ids,
                     const float* gates, int64_t r0, int64_t r1, float* y /* batch x (r1-r0) */);

typedef struct {
    int64_t rank, grid_rows, grid_cols;
    const uint16_t* placement;   /* K x 2 (p, q)                               */
    const int8_t* u_codes;       /* M x o x r                                  */
    const float* u_absmax;       /* M                                          */
    const int8_t* v_codes;       /* N x r x i                                  */
    const float* v_absmax;       /* N                                          */
    const uint16_t* singulars;   /* r binary16                                 */
    const float* scaling;        /* K x i                                      */
} tqo_tiled;

int tqo_lotile_forward(const float* x, int64_t batch, int64_t in_dim, int64_t out_dim,
                       int64_t num_experts, int64_t top_k, const tqo_tiled* t,
                       const int64_t* ids, const float* gates, int64_t r0, int64_t r1,
                       float* y /* batch x (r1-r0) */);

/* spd_inverse (quant.cpp:72-112): Cholesky H = L L^T, L^-1 by columns,
 * Hinv = L^-T L^-1, every dot in the reference's loop order.  h: n x n f32,
 * hinv: n x n f64.  Returns 0, or 6 (NumericError) with *bad_col / *bad_pivot
 * set at the first non-positive or non-finite pivot. */
int tqo_spd_inverse(const float* h, int64_t n, double* hinv, int64_t* bad_col, double* bad_pivot);

#ifdef __cplusplus
}
#endif
#endif
