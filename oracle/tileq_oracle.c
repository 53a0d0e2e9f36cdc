/* TEST INFRASTRUCTURE ONLY -- the checker, never the product.
 * Plain-C restatement of the reference hot path; see tileq_oracle.h.
 * Built with -ffp-contract=off so every double product/sum rounds exactly
 * as the reference's x86-64 build (no FMA contraction) does.
 */
#include "tileq_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- codec -- */

static float f32_of(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }
static uint32_t bits_of(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }

/* half_bits_to_float, codec.cpp:70-90 */
float tqo_half_to_float(uint16_t bits) {
    uint32_t sign = (uint32_t)(bits & 0x8000u) << 16;
    uint32_t exp = (bits >> 10) & 0x1Fu;
    uint32_t mant = bits & 0x3FFu;
    if (exp == 0x1Fu) return f32_of(sign | 0x7F800000u | (mant << 13));
    if (exp != 0) return f32_of(sign | ((exp + 112u) << 23) | (mant << 13));
    if (mant == 0) return f32_of(sign);
    uint32_t e = 113;
    while ((mant & 0x400u) == 0) { mant <<= 1; --e; }
    mant &= 0x3FFu;
    return f32_of(sign | (e << 23) | (mant << 13));
}

static uint32_t rne_bump(uint32_t base, uint32_t rem, uint32_t half) {
    if (rem > half || (rem == half && (base & 1u))) return base + 1u;
    return base;
}

/* float_to_half_bits, codec.cpp:38-68 */
uint16_t tqo_float_to_half(float value) {
    uint32_t u = bits_of(value);
    uint16_t sign = (uint16_t)((u >> 16) & 0x8000u);
    int32_t exp = (int32_t)((u >> 23) & 0xFFu) - 127;
    uint32_t mant = u & 0x7FFFFFu;
    if (exp == 128) return (uint16_t)(sign | (mant ? 0x7E00u : 0x7C00u));
    if (exp > 15) return (uint16_t)(sign | 0x7C00u);
    if (exp >= -14) {
        uint32_t base = ((uint32_t)(exp + 15) << 10) | (mant >> 13);
        base = rne_bump(base, mant & 0x1FFFu, 0x1000u);
        return (uint16_t)(sign | base);
    }
    if (exp < -25) return sign;
    uint32_t full = 0x800000u | mant;
    int shift = -exp - 1;
    uint32_t base = full >> shift;
    uint32_t dropped = full & ((1u << shift) - 1u);
    base = rne_bump(base, dropped, 1u << (shift - 1));
    return (uint16_t)(sign | base);
}

static int width_ok(int bits) { return bits == 2 || bits == 3 || bits == 4 || bits == 8; }

/* packed_byte_length, codec.cpp:145-148 */
int64_t tqo_packed_byte_length(int64_t count, int bits) {
    if (!width_ok(bits)) return -1;
    return (count * bits + 7) / 8;
}

/* pack_codes, codec.cpp:150-166: code t occupies stream bits [t*b, (t+1)*b), LSB-first */
int tqo_pack_codes(const uint32_t* codes, int64_t count, int bits, uint8_t* out) {
    if (!width_ok(bits)) return TQO_PARAM;
    int64_t nbytes = tqo_packed_byte_length(count, bits);
    memset(out, 0, (size_t)nbytes);
    int64_t bitpos = 0;
    for (int64_t t = 0; t < count; ++t) {
        uint32_t c = codes[t];
        if (c >= (1u << bits)) return TQO_PARAM;
        for (int b = 0; b < bits; ++b, ++bitpos)
            if (c & (1u << b)) out[bitpos >> 3] |= (uint8_t)(1u << (bitpos & 7));
    }
    return TQO_OK;
}

/* unpack_codes, codec.cpp:168-195 (incl. the nonzero-padding FormatError) */
int tqo_unpack_codes(const uint8_t* bytes, int64_t nbytes, int bits, int64_t count, uint32_t* out) {
    if (!width_ok(bits)) return TQO_PARAM;
    if (nbytes != tqo_packed_byte_length(count, bits)) return TQO_PARAM;
    int64_t bitpos = 0;
    for (int64_t t = 0; t < count; ++t) {
        uint32_t c = 0;
        for (int b = 0; b < bits; ++b, ++bitpos)
            if (bytes[bitpos >> 3] & (1u << (bitpos & 7))) c |= 1u << b;
        out[t] = c;
    }
    for (; bitpos < nbytes * 8; ++bitpos)
        if (bytes[bitpos >> 3] & (1u << (bitpos & 7))) return TQO_FORMAT;
    return TQO_OK;
}

/* zlib crc32_z(0, ...) as used by io.cpp:71-75 (reflected poly 0xEDB88320) */
uint32_t tqo_crc32(const uint8_t* data, int64_t n) {
    static uint32_t table[256];
    static int init = 0;
    if (!init) {
        for (uint32_t i = 0; i < 256; ++i) {
            uint32_t c = i;
            for (int k = 0; k < 8; ++k) c = (c & 1u) ? 0xEDB88320u ^ (c >> 1) : c >> 1;
            table[i] = c;
        }
        init = 1;
    }
    uint32_t crc = 0xFFFFFFFFu;
    for (int64_t t = 0; t < n; ++t) crc = table[(crc ^ data[t]) & 0xFFu] ^ (crc >> 8);
    return crc ^ 0xFFFFFFFFu;
}

/* ---------------------------------------------------------------- dequant -- */

static uint32_t code_at(const uint8_t* packed, int bits, int64_t t) {
    int64_t bitpos = t * bits;
    uint32_t c = 0;
    for (int b = 0; b < bits; ++b, ++bitpos)
        if (packed[bitpos >> 3] & (1u << (bitpos & 7))) c |= 1u << b;
    return c;
}

/* dequantize scalar mode, quant.cpp:289-302:
 * W[r,c] = float(double(code - zero) * scale), grid = grids[r*groups + c/g] */
int tqo_dequantize_rows(const tqo_qmat* q, int64_t out_dim, int64_t in_dim, int64_t r0,
                        int64_t r1, float* out) {
    if (!width_ok(q->bits) || q->group_size < 1) return TQO_PARAM;
    int64_t groups = (in_dim + q->group_size - 1) / q->group_size;
    for (int64_t r = r0; r < r1; ++r) {
        for (int64_t c = 0; c < in_dim; ++c) {
            int64_t g = r * groups + c / q->group_size;
            int64_t code = (int64_t)code_at(q->packed, q->bits, r * in_dim + c);
            float scale = tqo_half_to_float(q->scales[g]);
            out[(r - r0) * in_dim + c] = (float)((double)(code - (int64_t)q->zeros[g]) * scale);
        }
    }
    (void)out_dim;
    return TQO_OK;
}

/* ---------------------------------------------------------------- route -- */

/* route, moe.cpp:43-89.  scores = matmul(x, G^T) (matrix.cpp:25-36: one f64
 * dot in index order, rounded once); f64 max-subtracted softmax over all K;
 * order by (prob desc, index asc); gates = float(prob / selected_sum). */
int tqo_route(const float* x, int64_t batch, int64_t in_dim, const float* gate,
              int64_t num_experts, int64_t top_k, int64_t* ids, float* gates) {
    if (top_k < 1 || top_k > num_experts) return TQO_PARAM;
    float* scores = (float*)malloc(sizeof(float) * (size_t)num_experts);
    double* prob = (double*)malloc(sizeof(double) * (size_t)num_experts);
    int64_t* order = (int64_t*)malloc(sizeof(int64_t) * (size_t)num_experts);
    for (int64_t b = 0; b < batch; ++b) {
        const float* xb = x + b * in_dim;
        for (int64_t k = 0; k < num_experts; ++k) {
            const float* gk = gate + k * in_dim;
            double acc = 0.0;
            for (int64_t c = 0; c < in_dim; ++c) acc += (double)xb[c] * (double)gk[c];
            scores[k] = (float)acc;
        }
        double mx = scores[0];
        for (int64_t k = 1; k < num_experts; ++k) mx = fmax(mx, (double)scores[k]);
        double total = 0.0;
        for (int64_t k = 0; k < num_experts; ++k) {
            prob[k] = exp((double)scores[k] - mx);
            total += prob[k];
        }
        for (int64_t k = 0; k < num_experts; ++k) prob[k] /= total;
        /* selection of the top_k by (prob desc, index asc): equivalent to the
         * reference's full std::sort with that comparator (a strict total order) */
        for (int64_t k = 0; k < num_experts; ++k) order[k] = k;
        for (int64_t t = 0; t < top_k; ++t) {
            int64_t best = t;
            for (int64_t k = t + 1; k < num_experts; ++k) {
                int64_t a = order[k], c = order[best];
                if (prob[a] > prob[c] || (prob[a] == prob[c] && a < c)) best = k;
            }
            int64_t tmp = order[t]; order[t] = order[best]; order[best] = tmp;
        }
        double selected = 0.0;
        for (int64_t t = 0; t < top_k; ++t) selected += prob[order[t]];
        for (int64_t t = 0; t < top_k; ++t) {
            ids[b * top_k + t] = order[t];
            gates[b * top_k + t] = (float)(prob[order[t]] / selected);
        }
    }
    free(scores); free(prob); free(order);
    return TQO_OK;
}

/* ---------------------------------------------------------------- permute -- */

/* Token permutation (no reference counterpart):
 * pairs f = b*top_k + t, stable counting sort by ids[f] (experts ascending,
 * f ascending within an expert).  offsets = exclusive prefix of counts
 * (K+1 entries), perm[pos] = f, inv[f] = pos. */
int tqo_permute(const int64_t* ids, int64_t batch, int64_t top_k, int64_t num_experts,
                int32_t* perm, int32_t* offsets, int32_t* inv) {
    int64_t n = batch * top_k;
    for (int64_t e = 0; e <= num_experts; ++e) offsets[e] = 0;
    for (int64_t f = 0; f < n; ++f) {
        if (ids[f] < 0 || ids[f] >= num_experts) return TQO_PARAM;
        offsets[ids[f] + 1]++;
    }
    for (int64_t e = 0; e < num_experts; ++e) offsets[e + 1] += offsets[e];
    int32_t* cursor = (int32_t*)malloc(sizeof(int32_t) * (size_t)(num_experts + 1));
    memcpy(cursor, offsets, sizeof(int32_t) * (size_t)(num_experts + 1));
    for (int64_t f = 0; f < n; ++f) {
        int32_t pos = cursor[ids[f]]++;
        perm[pos] = (int32_t)f;
        inv[f] = pos;
    }
    free(cursor);
    return TQO_OK;
}

/* ---------------------------------------------------------------- qmoe -- */

/* qmoe_forward, infer.cpp:40-51 == reference_forward (moe.cpp:91-135) over
 * dequantize()d experts: out[b,r] = float( sum_t double(g_bt) * sum_c
 * double(W_e[r,c]) * x[b,c]  +  sum_s sum_c W_s[r,c] * x[b,c] ), t ascending
 * then shared, one f64 accumulator per output element.  Rows r in [r0, r1). */
int tqo_qmoe_forward(const float* x, int64_t batch, int64_t in_dim, int64_t out_dim,
                     int64_t num_experts, int64_t num_shared, int64_t top_k,
                     const tqo_qmat* experts, const int64_t* ids, const float* gates,
                     int64_t r0, int64_t r1, float* y) {
    float* wrow = (float*)malloc(sizeof(float) * (size_t)in_dim);
    int64_t nr = r1 - r0;
    for (int64_t b = 0; b < batch; ++b) {
        for (int64_t t = 0; t < top_k; ++t)
            if (ids[b * top_k + t] < 0 || ids[b * top_k + t] >= num_experts) { free(wrow); return TQO_PARAM; }
    }
    for (int64_t r = r0; r < r1; ++r) {
        for (int64_t b = 0; b < batch; ++b) {
            const float* xb = x + b * in_dim;
            double acc = 0.0;
            for (int64_t t = 0; t < top_k; ++t) {
                int64_t e = ids[b * top_k + t];
                double g = (double)gates[b * top_k + t];
                tqo_dequantize_rows(&experts[e], out_dim, in_dim, r, r + 1, wrow);
                double dot = 0.0;
                for (int64_t c = 0; c < in_dim; ++c) dot += (double)wrow[c] * (double)xb[c];
                acc += g * dot;
            }
            for (int64_t s = 0; s < num_shared; ++s) {
                tqo_dequantize_rows(&experts[num_experts + s], out_dim, in_dim, r, r + 1, wrow);
                double dot = 0.0;
                for (int64_t c = 0; c < in_dim; ++c) dot += (double)wrow[c] * (double)xb[c];
                acc += dot;
            }
            y[b * nr + (r - r0)] = (float)acc;
        }
    }
    free(wrow);
    return TQO_OK;
}

/* ---------------------------------------------------------------- lotile -- */

enum { TIER_FOLDED = 0, TIER_SCALAR = 1, TIER_GENERAL = 2 };

/* lotile_forward, infer.cpp:53-180, restated step by step. */
int tqo_lotile_forward(const float* x, int64_t batch, int64_t in_dim, int64_t out_dim,
                       int64_t num_experts, int64_t top_k, const tqo_tiled* t,
                       const int64_t* ids, const float* gates, int64_t r0, int64_t r1,
                       float* y) {
    const int64_t m = t->grid_rows, n = t->grid_cols, r = t->rank, i = in_dim, o = out_dim;
    /* placement bounds (infer.cpp:65-72) */
    for (int64_t k = 0; k < num_experts; ++k)
        if (t->placement[2 * k] >= m || t->placement[2 * k + 1] >= n) return TQO_FORMAT;

    /* decoded factor values: value = float(code) * (absmax / 127.0f) (codec.cpp:122-129) */
    float* sig = (float*)malloc(sizeof(float) * (size_t)r);
    for (int64_t j = 0; j < r; ++j) sig[j] = tqo_half_to_float(t->singulars[j]);

    /* tier per column block (infer.cpp:74-99) */
    int* tier = (int*)malloc(sizeof(int) * (size_t)n);
    int64_t* first = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
    for (int64_t q = 0; q < n; ++q) {
        int any = 0, all_same = 1, all_scalar = 1;
        first[q] = -1;
        for (int64_t k = 0; k < num_experts; ++k) {
            if (t->placement[2 * k + 1] != q) continue;
            const float* sk = t->scaling + k * i;
            if (!any) { first[q] = k; any = 1; }
            else if (memcmp(sk, t->scaling + first[q] * i, sizeof(float) * (size_t)i) != 0) {
                /* std::vector<float> operator!= compares with ==, so -0/+0
                 * and NaN differ from memcmp only for values the quantizer
                 * never produces (scalings are strictly positive) */
                all_same = 0;
            }
            for (int64_t c = 0; c < i; ++c) if (sk[c] != sk[0]) { all_scalar = 0; break; }
        }
        if (!any || all_same) tier[q] = TIER_FOLDED;
        else if (all_scalar) tier[q] = TIER_SCALAR;
        else tier[q] = TIER_GENERAL;
    }

    /* stacked projection P ((N*r) x i), infer.cpp:104-117 */
    float* proj = (float*)malloc(sizeof(float) * (size_t)(n * r * i));
    for (int64_t q = 0; q < n; ++q) {
        const float vscale = t->v_absmax[q] == 0.0f ? 0.0f : t->v_absmax[q] / 127.0f;
        for (int64_t j = 0; j < r; ++j) {
            const double sigma = sig[j];
            for (int64_t c = 0; c < i; ++c) {
                float v = (float)t->v_codes[(q * r + j) * i + c] * vscale;
                double val = sigma * (double)v;
                if (tier[q] == TIER_FOLDED && first[q] >= 0) val /= t->scaling[first[q] * i + c];
                proj[(q * r + j) * i + c] = (float)val;
            }
        }
    }

    /* GEMM 1: x_proj = float(f64 x . P^T), infer.cpp:121 */
    float* xproj = (float*)malloc(sizeof(float) * (size_t)(batch * n * r));
    for (int64_t b = 0; b < batch; ++b)
        for (int64_t col = 0; col < n * r; ++col) {
            double acc = 0.0;
            for (int64_t c = 0; c < i; ++c)
                acc += (double)x[b * i + c] * (double)proj[col * i + c];
            xproj[b * n * r + col] = (float)acc;
        }

    /* gather / gate / scatter, infer.cpp:125-157 */
    double* sacc = (double*)calloc((size_t)(batch * m * r), sizeof(double));
    double* descaled = (double*)malloc(sizeof(double) * (size_t)i);
    for (int64_t b = 0; b < batch; ++b) {
        for (int64_t tt = 0; tt < top_k; ++tt) {
            int64_t e = ids[b * top_k + tt];
            double g = (double)gates[b * top_k + tt];
            int64_t p = t->placement[2 * e], q = t->placement[2 * e + 1];
            double* dst = sacc + (b * m + p) * r;
            if (tier[q] == TIER_FOLDED) {
                for (int64_t j = 0; j < r; ++j) dst[j] += g * (double)xproj[b * n * r + q * r + j];
            } else if (tier[q] == TIER_SCALAR) {
                double inv = 1.0 / t->scaling[e * i];
                for (int64_t j = 0; j < r; ++j) dst[j] += g * ((double)xproj[b * n * r + q * r + j] * inv);
            } else {
                const float* sk = t->scaling + e * i;
                for (int64_t c = 0; c < i; ++c) descaled[c] = (double)x[b * i + c] / sk[c];
                for (int64_t j = 0; j < r; ++j) {
                    const float* prow = proj + (q * r + j) * i;
                    double acc = 0.0;
                    for (int64_t c = 0; c < i; ++c) acc += (double)prow[c] * descaled[c];
                    dst[j] += g * acc;
                }
            }
        }
    }

    /* s_buf = float(s_acc); GEMM 2 against U_flat[p*r+j, c] = u_p[c, j], infer.cpp:158-174 */
    int64_t nrow = r1 - r0;
    for (int64_t b = 0; b < batch; ++b) {
        for (int64_t c = r0; c < r1; ++c) {
            double acc = 0.0;
            for (int64_t p = 0; p < m; ++p) {
                const float uscale = t->u_absmax[p] == 0.0f ? 0.0f : t->u_absmax[p] / 127.0f;
                for (int64_t j = 0; j < r; ++j) {
                    float s = (float)sacc[(b * m + p) * r + j];
                    float u = (float)t->u_codes[(p * o + c) * r + j] * uscale;
                    acc += (double)s * (double)u;
                }
            }
            y[b * nrow + (c - r0)] = (float)acc;
        }
    }
    free(sig); free(tier); free(first); free(proj); free(xproj); free(sacc); free(descaled);
    return TQO_OK;
}

/* ------------------------------------------------------ producer: spd_inverse -- */

/* quant.cpp:72-112, loop for loop */
int tqo_spd_inverse(const float* h, int64_t n, double* hinv, int64_t* bad_col, double* bad_pivot) {
    double* chol = (double*)calloc((size_t)(n * n), sizeof(double));
    double* linv = (double*)calloc((size_t)(n * n), sizeof(double));
    if (!chol || !linv) { free(chol); free(linv); return 99; }
    for (int64_t j = 0; j < n; ++j) {
        for (int64_t i = j; i < n; ++i) {
            double acc = (double)h[i * n + j];
            for (int64_t k = 0; k < j; ++k) acc -= chol[i * n + k] * chol[j * n + k];
            if (i == j) {
                if (acc <= 0.0 || !isfinite(acc)) {
                    *bad_col = j;
                    *bad_pivot = acc;
                    free(chol); free(linv);
                    return 6;
                }
                chol[i * n + j] = sqrt(acc);
            } else {
                chol[i * n + j] = acc / chol[j * n + j];
            }
        }
    }
    for (int64_t j = 0; j < n; ++j) {
        linv[j * n + j] = 1.0 / chol[j * n + j];
        for (int64_t i = j + 1; i < n; ++i) {
            double acc = 0.0;
            for (int64_t k = j; k < i; ++k) acc += chol[i * n + k] * linv[k * n + j];
            linv[i * n + j] = -acc / chol[i * n + i];
        }
    }
    for (int64_t i = 0; i < n; ++i) {
        for (int64_t j = 0; j <= i; ++j) {
            double acc = 0.0;
            for (int64_t k = i; k < n; ++k) acc += linv[k * n + i] * linv[k * n + j];
            hinv[i * n + j] = acc;
            hinv[j * n + i] = acc;
        }
    }
    free(chol);
    free(linv);
    return 0;
}
