// Host runtime of libtileq_b200.so: artifact loader (validation identical to
// the reference read_artifact, io.cpp:679-813), repack of the packed weights
// into the engine's TMA tile layout, device workspace, and the C-ABI entry
// points declared in include/tileq_b200.h.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <memory>
#include <set>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <json.hpp>
#include <zlib.h>

#include "../../include/tileq_b200.h"
#include "tq_internal.h"

namespace fs = std::filesystem;
using nlohmann::json;

namespace tqb {

// launch wrappers (tq_kernels.cu)
cudaError_t launch_gemm(const GemmParams& p, int grid, cudaStream_t stream);
cudaError_t launch_route(const float* x, int batch, int in_dim, const float* gate, int num_experts, int top_k,
                         int group_size, int groups, int k_pad, int32_t* ids, float* gates, __half* x16, float* sx,
                         float* score_ws, int32_t* ticket,
                         cudaStream_t stream);
cudaError_t launch_plan(const PlanArgs& a, cudaStream_t stream);
cudaError_t launch_gather(const GatherArgs& a, int max_rows, cudaStream_t stream);
cudaError_t launch_gather_tokens(const GatherArgs& a, cudaStream_t stream);
cudaError_t launch_combine(const CombineArgs& a, cudaStream_t stream);
cudaError_t launch_lr_right(const float* A, int64_t a_ld, int rows, const float* x, int64_t x_ld, int tokens, int n,
                            const float* scale, float* mid, int64_t mid_ld, cudaStream_t stream);
cudaError_t launch_lr_left(const float* U, int o, int r, const float* mid, const float* gate, float* acc,
                           cudaStream_t stream);
cudaError_t launch_dequant_all(const DequantAllArgs& a, int bits, cudaStream_t stream);
cudaError_t launch_unpack(const uint8_t* bytes, int64_t nbytes, int bits, int64_t count, uint32_t* out,
                          int32_t* err_flag, cudaStream_t stream);
cudaError_t launch_dec_route(const DecRouteArgs& a, cudaStream_t stream);
cudaError_t launch_dec_combine(const DecCombineArgs& a, cudaStream_t stream);
cudaError_t launch_decode(const DecParams& p, int dn, int grid, cudaStream_t stream);
cudaError_t launch_export_codes(const uint8_t* wcodes, int bits, int kc_total, int out_dim, int in_dim,
                                uint32_t* out, cudaStream_t stream);
cudaError_t launch_exp_f64(const double* x, int64_t n, double* y, cudaStream_t stream);
cudaError_t launch_repack_codes(const uint8_t* packed, int64_t nbytes, int bits, int64_t o, int64_t i,
                                int64_t mb_count, int64_t kc_total, uint8_t* out, cudaStream_t stream);
// artifact producer (tq_producer.cu)
cudaError_t launch_estimate_hessian(const float* x, int64_t tokens, int64_t dim, double damping, double* acc,
                                    double* lambda, float* h, cudaStream_t stream);
size_t spd_status_bytes();
cudaError_t launch_spd_inverse(const float* h, int64_t n, double* chol, double* linv, double* hinv, void* status,
                               cudaStream_t stream);
void spd_status_read(const void* host_copy, int* failed, int64_t* column, double* pivot);
cudaError_t launch_make_grids(const float* r, int64_t rows, int64_t cols, int bits, int64_t gs, float* scales,
                              int32_t* zeros, cudaStream_t stream);
cudaError_t launch_rtn_codes(const float* r, int64_t rows, int64_t cols, int bits, int64_t gs, const float* scales,
                             const int32_t* zeros, uint8_t* codes, cudaStream_t stream);
int gptq_rows_per_cta(int64_t dim, int64_t gs);
cudaError_t launch_gptq(const float* r, int64_t rows, int64_t dim, int bits, int64_t gs, const float* scales,
                        const int32_t* zeros, const double* hinv, uint8_t* codes, cudaStream_t stream);
cudaError_t launch_proxy_loss(const float* orig, const uint8_t* codes, const float* scales, const int32_t* zeros,
                              int64_t rows, int64_t dim, int64_t gs, const float* h, int64_t chunk_rows, double* he_t,
                              double* rowsum, double* total, cudaStream_t stream);
cudaError_t launch_widen(const float* w, int64_t n, double* out, cudaStream_t stream);
cudaError_t launch_matvec(const double* a, int64_t rows, int64_t cols, const double* x, double* y,
                          cudaStream_t stream);
cudaError_t launch_mattvec(const double* a, int64_t rows, int64_t cols, const double* x, double* y,
                           cudaStream_t stream);
cudaError_t launch_norm2(const double* v, int64_t n, double* out, cudaStream_t stream);
cudaError_t launch_div_by(const double* src, int64_t n, const double* d, double* dst, cudaStream_t stream);
cudaError_t launch_deflate(double* a, int64_t rows, int64_t cols, const double* sigma, const double* u,
                           const double* v, cudaStream_t stream);
cudaError_t launch_pack_triples(const double* us, const double* vs, const int32_t* order, int64_t rank, int64_t rows,
                                int64_t cols, float* left, float* right, cudaStream_t stream);
cudaError_t launch_ep_units(const int32_t* counts, int n_src, int e_stride, int n_local, int slab, int mb_count, int bn,
                            int kc_end, int n_ext, Unit* units, int32_t* n_units, cudaStream_t stream);

// ---------------------------------------------------------------------------
// errors
// ---------------------------------------------------------------------------

struct TqError : std::runtime_error {
    tq_status code;
    TqError(tq_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

thread_local std::string g_last_error;

[[noreturn]] void fail(tq_status c, const std::string& m) { throw TqError(c, m); }

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) fail(TQ_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

template <class F>
tq_status guarded(F&& body) {
    try {
        body();
        return TQ_OK;
    } catch (const TqError& e) {
        g_last_error = e.what();
        return e.code;
    } catch (const std::bad_alloc&) {
        g_last_error = "host allocation failed";
        return TQ_ERR_SIZE;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return TQ_ERR_INTERNAL;
    }
}

// ---------------------------------------------------------------------------
// binary16 helpers (codec.cpp:38-92 semantics)
// ---------------------------------------------------------------------------

float half_bits_to_float(uint16_t bits) {
    const uint32_t sign = static_cast<uint32_t>(bits & 0x8000u) << 16;
    const uint32_t exp = (bits >> 10) & 0x1Fu;
    uint32_t mant = bits & 0x3FFu;
    uint32_t u;
    if (exp == 0x1Fu) {
        u = sign | 0x7F800000u | (mant << 13);
    } else if (exp != 0) {
        u = sign | ((exp + 112u) << 23) | (mant << 13);
    } else if (mant == 0) {
        u = sign;
    } else {
        uint32_t e = 113;
        while ((mant & 0x400u) == 0) {
            mant <<= 1;
            --e;
        }
        u = sign | (e << 23) | ((mant & 0x3FFu) << 13);
    }
    float f;
    std::memcpy(&f, &u, 4);
    return f;
}

uint16_t float_to_half_bits(float value) {
    // round-to-nearest-even; used for values that are exactly representable
    // (scaled scales, small integers) and for the fp16 projection weights
    const __half h = __float2half_rn(value);
    uint16_t b;
    std::memcpy(&b, &h, 2);
    return b;
}

// ---------------------------------------------------------------------------
// artifact container reader (io.cpp:186-295 semantics)
// ---------------------------------------------------------------------------

size_t packed_byte_length(size_t count, int bits) { return (count * static_cast<size_t>(bits) + 7) / 8; }

bool packed_dtype(const std::string& dt, int* bits) {
    for (int b : {2, 3, 4, 8})
        if (dt == "packed-u" + std::to_string(b)) {
            if (bits) *bits = b;
            return true;
        }
    return false;
}

size_t expected_bytes(const std::vector<size_t>& shape, const std::string& dtype) {
    size_t n = 1;
    for (size_t d : shape) {
        if (d != 0 && n > SIZE_MAX / d) fail(TQ_ERR_FORMAT, "tensor shape overflows element count");
        n *= d;
    }
    int bits = 0;
    if (packed_dtype(dtype, &bits)) return packed_byte_length(n, bits);
    if (dtype == "f32") return n * 4;
    if (dtype == "f16-roundtrip" || dtype == "u16") return n * 2;
    if (dtype == "u8") return n;
    fail(TQ_ERR_FORMAT, "unknown tensor dtype '" + dtype + "'");
}

class Container {
   public:
    Container(const std::string& dir, bool verify) : dir_(dir), verify_(verify) {
        const fs::path path = fs::path(dir) / "manifest.json";
        std::ifstream in(path, std::ios::binary);
        if (!in) fail(TQ_ERR_IO, "cannot open '" + path.string() + "'");
        std::string text((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
        try {
            m_ = json::parse(text);
        } catch (const json::parse_error& e) {
            fail(TQ_ERR_FORMAT, std::string("manifest is not valid JSON: ") + e.what());
        }
        if (!m_.is_object() || !m_.contains("format_version") || !m_["format_version"].is_number_integer())
            fail(TQ_ERR_FORMAT, "manifest missing integer format_version");
        const int version = m_["format_version"].get<int>();
        if (version != 1)
            fail(TQ_ERR_FORMAT,
                 "unsupported container format_version " + std::to_string(version) + " (expected 1)");
        const std::string kind = m_.value("kind", std::string());
        if (kind != "tileq_artifact")
            fail(TQ_ERR_FORMAT, "expected a 'tileq_artifact' container, found '" + kind + "'");
        if (!m_.contains("tensors") || !m_["tensors"].is_object())
            fail(TQ_ERR_FORMAT, "manifest missing tensors object");
        if (!m_.contains("meta") || !m_["meta"].is_object()) fail(TQ_ERR_FORMAT, "manifest missing meta object");
    }

    const json& meta() const { return m_["meta"]; }

    std::vector<uint8_t> bytes(const std::string& name, const std::string& dtype,
                               std::vector<size_t>* shape_out = nullptr) const {
        const json& tensors = m_["tensors"];
        if (!tensors.contains(name)) fail(TQ_ERR_FORMAT, "missing tensor '" + name + "'");
        const json& e = tensors[name];
        if (!e.is_object() || !e.contains("shape") || !e.contains("dtype") || !e.contains("byte_length") ||
            !e.contains("crc32") || !e.contains("file"))
            fail(TQ_ERR_FORMAT, "tensor '" + name + "': malformed manifest entry");
        const std::string actual = e["dtype"].get<std::string>();
        if (actual != dtype)
            fail(TQ_ERR_FORMAT, "tensor '" + name + "': dtype is '" + actual + "', expected '" + dtype + "'");
        std::vector<size_t> shape = e["shape"].get<std::vector<size_t>>();
        const size_t declared = e["byte_length"].get<size_t>();
        if (expected_bytes(shape, dtype) != declared)
            fail(TQ_ERR_FORMAT, "tensor '" + name + "': byte_length does not match shape/dtype");
        const fs::path path = fs::path(dir_) / e["file"].get<std::string>();
        std::error_code ec;
        const auto on_disk = fs::file_size(path, ec);
        if (ec) fail(TQ_ERR_IO, "tensor '" + name + "': cannot stat '" + path.string() + "'");
        if (on_disk != declared)
            fail(TQ_ERR_FORMAT, "tensor '" + name + "': blob is " + std::to_string(on_disk) +
                                    " bytes, manifest says " + std::to_string(declared));
        std::ifstream in(path, std::ios::binary);
        if (!in) fail(TQ_ERR_IO, "tensor '" + name + "': cannot open '" + path.string() + "'");
        std::vector<uint8_t> data(declared);
        in.read(reinterpret_cast<char*>(data.data()), static_cast<std::streamsize>(declared));
        if (static_cast<size_t>(in.gcount()) != declared)
            fail(TQ_ERR_IO, "tensor '" + name + "': short read from '" + path.string() + "'");
        if (verify_) {
            const uint32_t want = e["crc32"].get<uint32_t>();
            uLong crc = crc32_z(0L, Z_NULL, 0);
            crc = crc32_z(crc, data.data(), data.size());
            if (static_cast<uint32_t>(crc) != want) fail(TQ_ERR_FORMAT, "tensor '" + name + "': checksum mismatch");
        }
        if (shape_out) *shape_out = std::move(shape);
        return data;
    }

   private:
    std::string dir_;
    bool verify_;
    json m_;
};

const json& require_object(const json& j, const char* key) {
    if (!j.contains(key) || !j[key].is_object())
        fail(TQ_ERR_FORMAT, "manifest meta missing object '" + std::string(key) + "'");
    return j[key];
}

size_t require_size(const json& j, const char* key) {
    if (!j.contains(key) || !j[key].is_number_unsigned())
        fail(TQ_ERR_FORMAT, "manifest meta missing unsigned field '" + std::string(key) + "'");
    return j[key].get<size_t>();
}

std::string require_string(const json& j, const char* key) {
    if (!j.contains(key) || !j[key].is_string())
        fail(TQ_ERR_FORMAT, "manifest meta missing string field '" + std::string(key) + "'");
    return j[key].get<std::string>();
}

// One quantized matrix as read from the wire (read_quantized, io.cpp:422-485).
struct QMat {
    int bits = 0;
    bool vec = false;              // codebook (vector) mode
    size_t gs = 0;                 // scalar mode group size
    size_t sub_dim = 0;            // vector mode subvector length
    std::vector<uint16_t> codebook;   // 2^bits x sub_dim binary16 (vector mode)
    std::vector<uint8_t> packed;
    std::vector<uint16_t> scales;  // o x G binary16
    std::vector<uint8_t> zeros;    // o x G unpacked
};

std::vector<uint32_t> unpack_stream(const std::vector<uint8_t>& bytes, int bits, size_t count, const std::string& what) {
    if (bytes.size() != packed_byte_length(count, bits))
        fail(TQ_ERR_FORMAT, what + ": packed stream length mismatch");
    std::vector<uint32_t> out(count);
    const uint32_t mask = (1u << bits) - 1u;
    for (size_t t = 0; t < count; ++t) {
        const size_t bit = t * static_cast<size_t>(bits);
        uint32_t w = bytes[bit >> 3];
        if ((bit >> 3) + 1 < bytes.size()) w |= static_cast<uint32_t>(bytes[(bit >> 3) + 1]) << 8;
        out[t] = (w >> (bit & 7)) & mask;
    }
    for (size_t bit = count * static_cast<size_t>(bits); bit < bytes.size() * 8; ++bit)
        if (bytes[bit >> 3] & (1u << (bit & 7)))
            fail(TQ_ERR_FORMAT, what + ": packed stream has nonzero padding past code " + std::to_string(count));
    return out;
}

// length and clean trailing pad bits of a packed stream without unpacking it
// (unpack_codes' checks, codec.cpp:168-195)
void check_packed_stream(const std::vector<uint8_t>& bytes, int bits, size_t count, const std::string& what) {
    if (bytes.size() != packed_byte_length(count, bits)) fail(TQ_ERR_FORMAT, what + ": packed stream length mismatch");
    for (size_t bit = count * static_cast<size_t>(bits); bit < bytes.size() * 8; ++bit)
        if (bytes[bit >> 3] & (1u << (bit & 7)))
            fail(TQ_ERR_FORMAT, what + ": packed stream has nonzero padding past code " + std::to_string(count));
}

QMat read_qmat(const Container& c, const std::string& prefix, const json& qmeta, size_t o, size_t i) {
    int bits = 0;
    if (!qmeta.contains("bits") || !qmeta["bits"].is_number_integer() ||
        (bits = qmeta["bits"].get<int>(), bits != 2 && bits != 3 && bits != 4 && bits != 8))
        fail(TQ_ERR_FORMAT, "manifest quant meta: bits must be one of 2, 3, 4, 8");
    const std::string mode = require_string(qmeta, "mode");
    QMat q;
    q.bits = bits;
    std::vector<size_t> shape;
    if (mode == "vector") {
        // codebook mode (io.cpp:464-480): codes o x subvectors, codebook 2^bits x sub_dim f16
        q.vec = true;
        q.sub_dim = require_size(qmeta, "sub_dim");
        if (q.sub_dim == 0) fail(TQ_ERR_FORMAT, "manifest quant meta: sub_dim must be >= 1");
        const size_t subs = (i + q.sub_dim - 1) / q.sub_dim;
        q.packed = c.bytes(prefix + ".codes", "packed-u" + std::to_string(bits), &shape);
        if (shape != std::vector<size_t>{o, subs}) fail(TQ_ERR_FORMAT, "tensor '" + prefix + ".codes': unexpected shape");
        const std::vector<uint8_t> bb = c.bytes(prefix + ".codebook", "f16-roundtrip", &shape);
        if (shape != std::vector<size_t>{size_t{1} << bits, q.sub_dim})
            fail(TQ_ERR_FORMAT, "tensor '" + prefix + ".codebook': unexpected shape");
        q.codebook.resize(bb.size() / 2);
        std::memcpy(q.codebook.data(), bb.data(), bb.size());
        // the trailing pad bits of the code stream must be clean (unpack_codes, codec.cpp:168-195)
        check_packed_stream(q.packed, bits, o * subs, "tensor '" + prefix + ".codes'");
        return q;
    }
    if (mode != "scalar") fail(TQ_ERR_FORMAT, "manifest quant meta: unknown mode '" + mode + "'");
    const size_t gs = require_size(qmeta, "group_size");
    if (gs == 0) fail(TQ_ERR_FORMAT, "manifest quant meta: group_size must be >= 1");
    q.gs = gs;
    const size_t groups = (i + gs - 1) / gs;
    q.packed = c.bytes(prefix + ".codes", "packed-u" + std::to_string(bits), &shape);
    if (shape != std::vector<size_t>{o, i}) fail(TQ_ERR_FORMAT, "tensor '" + prefix + ".codes': unexpected shape");
    const std::vector<uint8_t> sb = c.bytes(prefix + ".scales", "f16-roundtrip", &shape);
    if (shape != std::vector<size_t>{o, groups}) fail(TQ_ERR_FORMAT, "tensor '" + prefix + ".scales': unexpected shape");
    q.scales.resize(o * groups);
    std::memcpy(q.scales.data(), sb.data(), sb.size());
    const std::vector<uint8_t> zb = c.bytes(prefix + ".zeros", "packed-u" + std::to_string(bits), &shape);
    if (shape != std::vector<size_t>{o, groups}) fail(TQ_ERR_FORMAT, "tensor '" + prefix + ".zeros': unexpected shape");
    const std::vector<uint32_t> z = unpack_stream(zb, bits, o * groups, "tensor '" + prefix + ".zeros'");
    q.zeros.resize(z.size());
    for (size_t t = 0; t < z.size(); ++t) q.zeros[t] = static_cast<uint8_t>(z[t]);
    for (size_t t = 0; t < q.scales.size(); ++t) {
        const float s = half_bits_to_float(q.scales[t]);
        if (!(s > 0.0f) || !std::isfinite(s)) fail(TQ_ERR_FORMAT, "tensor '" + prefix + ".scales': non-positive scale");
    }
    // the residual code stream itself: length and clean padding (unpacked again by the repack)
    check_packed_stream(q.packed, bits, o * i, "tensor '" + prefix + ".codes'");
    return q;
}

// ---------------------------------------------------------------------------
// device memory
// ---------------------------------------------------------------------------

struct DBuf {
    void* p = nullptr;
    size_t n = 0;
    DBuf() = default;
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    ~DBuf() { reset(); }
    void reset() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    void alloc(size_t bytes) {
        reset();
        if (bytes == 0) bytes = 16;
        cuda_check(cudaMalloc(&p, bytes), "cudaMalloc");
        n = bytes;
    }
    void upload(const void* src, size_t bytes) {
        alloc(bytes);
        if (bytes) cuda_check(cudaMemcpy(p, src, bytes, cudaMemcpyHostToDevice), "cudaMemcpy H2D");
    }
    template <class T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode_fn() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void* ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        cuda_check(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q),
                   "cudaGetDriverEntryPoint(cuTensorMapEncodeTiled)");
        if (!ptr || q != cudaDriverEntryPointSuccess) fail(TQ_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
        fn = reinterpret_cast<EncodeTiledFn>(ptr);
    }
    return fn;
}

// fp16 row-major [rows, cols] tensor, box [box_rows, 64], 128-byte swizzle; rows
// `ld` elements apart (0: cols)
CUtensorMap make_map(void* base, uint64_t rows, uint64_t cols, uint32_t box_rows, uint64_t ld = 0) {
    CUtensorMap m;
    std::memset(&m, 0, sizeof(m));
    const cuuint64_t dims[2] = {cols, std::max<uint64_t>(rows, 1)};
    const cuuint64_t strides[1] = {(ld ? ld : cols) * 2};
    const cuuint32_t box[2] = {64, box_rows};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = get_encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, base, dims, strides, box, estr,
                                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                       CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) fail(TQ_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
    return m;
}

// ---------------------------------------------------------------------------
// repack: wire codes -> engine tile layout
// ---------------------------------------------------------------------------


struct Geometry {
    int64_t K, top_k, i, o, S, r, M, N;
    int bits;
    int64_t gs, G;
    int64_t k_pad, kc_total, o_pad, mb_count;
    int64_t n_ext, ext_cols;
};

// Power-of-two prescale k of a matrix (s' = s * 2^k, max s' <= 16) so code*s'
// stays comfortably inside fp16 range; the epilogue multiplies by 2^-k.
int prescale_exponent(const QMat& q) {
    float smax = 0.0f;
    for (uint16_t sb : q.scales) smax = std::max(smax, half_bits_to_float(sb));
    int k = 0;
    if (smax > 0.0f) {
        k = static_cast<int>(std::floor(std::log2(16.0 / smax)));
        k = std::max(-24, std::min(24, k));
        while (std::ldexp(static_cast<double>(smax), k) > 16.0) --k;
    }
    return k;
}

// Scale / zero slabs of one scalar matrix ([mb][group][row], scales prescaled by
// 2^k); its code blocks are repacked on the device from the packed stream
// (repack_codes_kernel) once the layer's device memory exists.
void repack_slabs(const QMat& q, const Geometry& g, uint16_t* scales_out, uint8_t* zeros_out, int* k_out) {
    const int k = prescale_exponent(q);
    *k_out = k;
    for (int64_t mb = 0; mb < g.mb_count; ++mb)
        for (int64_t gi = 0; gi < g.G; ++gi)
            for (int rl = 0; rl < kBM; ++rl) {
                const int64_t row = mb * kBM + rl;
                const size_t dst = static_cast<size_t>((mb * g.G + gi) * kBM + rl);
                if (row < g.o) {
                    const float sv = half_bits_to_float(q.scales[static_cast<size_t>(row * g.G + gi)]);
                    scales_out[dst] = float_to_half_bits(std::ldexp(sv, k));
                    zeros_out[dst] = q.zeros[static_cast<size_t>(row * g.G + gi)];
                } else {
                    scales_out[dst] = 0;
                    zeros_out[dst] = 0;
                }
            }
}

// Codebook residual -> dense fp16 blocks in the engine's [mb][kc] layout: word
// (h * 16 + j) of row r of a 64-K block holds columns 32 h + 2 j, + 1 (the layout of
// the extension / projection blocks).
// W[r, c] = codebook[code(r, c / sub_dim)][c % sub_dim] (dequantize, quant.cpp:303-321).
void repack_vq(const QMat& q, const Geometry& g, uint8_t* codes_out, uint16_t* scales_out, uint8_t* zeros_out,
               int* k_out) {
    const size_t sd = q.sub_dim, subs = (static_cast<size_t>(g.i) + sd - 1) / sd;
    const std::vector<uint32_t> codes = unpack_stream(q.packed, q.bits, static_cast<size_t>(g.o) * subs, "codes");
    *k_out = 0;
    auto val = [&](int64_t row, int64_t col) -> uint32_t {
        if (row >= g.o || col >= g.i) return 0u;
        const uint32_t c = codes[static_cast<size_t>(row) * subs + static_cast<size_t>(col) / sd];
        return q.codebook[static_cast<size_t>(c) * sd + static_cast<size_t>(col) % sd];
    };
    const int blk = code_block_bytes(kDenseBits);
    for (int64_t mb = 0; mb < g.mb_count; ++mb) {
        for (int64_t kc = 0; kc < g.kc_total; ++kc) {
            uint32_t* block = reinterpret_cast<uint32_t*>(codes_out + (mb * g.kc_total + kc) * blk);
            for (int h = 0; h < 2; ++h)
                for (int j = 0; j < 16; ++j)
                    for (int rl = 0; rl < kBM; ++rl) {
                        const int64_t row = mb * kBM + rl, c0 = kc * kKC + 32 * h + 2 * j;
                        block[(h * 16 + j) * kBM + rl] = val(row, c0) | (val(row, c0 + 1) << 16);
                    }
        }
        for (int64_t gi = 0; gi < g.G; ++gi)
            for (int rl = 0; rl < kBM; ++rl) {
                const size_t dst = static_cast<size_t>((mb * g.G + gi) * kBM + rl);
                scales_out[dst] = mb * kBM + rl < g.o ? 0x3C00u : 0u;   // 1.0
                zeros_out[dst] = 0;
            }
    }
}

// Scalar residual with a group size the super-word dequant cannot serve: W'[r, c] =
// fp16((code - zero) * scale * 2^k) (dequantize, quant.cpp:285-323, computed in f64,
// rounded once; k = prescale_exponent keeps |W'| <= 255 * 16), dense blocks in the
// engine layout; the epilogue multiplies by 2^-k; unit scales, no zero points left.
void repack_dense_scalar(const QMat& q, const Geometry& g, uint8_t* codes_out, uint16_t* scales_out,
                         uint8_t* zeros_out, int* k_out) {
    const std::vector<uint32_t> codes = unpack_stream(q.packed, q.bits, static_cast<size_t>(g.o * g.i), "codes");
    const int k = prescale_exponent(q);
    *k_out = k;
    const size_t G = (static_cast<size_t>(g.i) + q.gs - 1) / q.gs;
    auto val = [&](int64_t row, int64_t col) -> uint32_t {
        if (row >= g.o || col >= g.i) return 0u;
        const size_t gi = static_cast<size_t>(row) * G + static_cast<size_t>(col) / q.gs;
        const double w = (static_cast<double>(codes[static_cast<size_t>(row * g.i + col)]) - q.zeros[gi]) *
                         static_cast<double>(half_bits_to_float(q.scales[gi]));
        return float_to_half_bits(static_cast<float>(std::ldexp(w, k)));
    };
    const int blk = code_block_bytes(kDenseBits);
    for (int64_t mb = 0; mb < g.mb_count; ++mb) {
        for (int64_t kc = 0; kc < g.kc_total; ++kc) {
            uint32_t* block = reinterpret_cast<uint32_t*>(codes_out + (mb * g.kc_total + kc) * blk);
            for (int h = 0; h < 2; ++h)
                for (int j = 0; j < 16; ++j)
                    for (int rl = 0; rl < kBM; ++rl) {
                        const int64_t row = mb * kBM + rl, c0 = kc * kKC + 32 * h + 2 * j;
                        block[(h * 16 + j) * kBM + rl] = val(row, c0) | (val(row, c0 + 1) << 16);
                    }
        }
        for (int64_t gi = 0; gi < g.G; ++gi)
            for (int rl = 0; rl < kBM; ++rl) {
                const size_t dst = static_cast<size_t>((mb * g.G + gi) * kBM + rl);
                scales_out[dst] = mb * kBM + rl < g.o ? 0x3C00u : 0u;
                zeros_out[dst] = 0;
            }
    }
}

}  // namespace tqb

using namespace tqb;

// ---------------------------------------------------------------------------
// the layer
// ---------------------------------------------------------------------------

struct tq_layer {
    int device = 0;
    Geometry g{};
    int64_t e_begin = 0, e_end = 0;     // resident routed experts
    int64_t n_weights = 0;              // resident routed + shared
    int64_t tiers[3] = {0, 0, 0};
    // projection (stacked X.A matrices)
    int64_t NP = 0, proj_rows = 0, proj_o_pad = 0, proj_mb = 0;
    // device tables
    DBuf gate, codes, scales, ext_blocks, w_outscale;
    DBuf pcodes, p_outscale, pm_of, zscale, rowscale;
    int64_t weight_stride = 0, pweight_stride = 0;
    int64_t device_bytes = 0;
    // workspace
    int64_t cap = 0;
    DBuf route_ws, route_ticket, poffsets;   // router: per-(token, expert) certified scores, per-token tickets
    DBuf ids, gates, x16, sx, perm, inv, offsets, units, n_units, punits, n_punits, zpart, xperm, extperm, ypart,
        err_flag, xin, yout, nsplit_d, hids, hgates, ep_units, ep_nunits;
    int64_t ep_units_cap = 0;
    int64_t ypart_cap_floats = 0, zpart_cap_floats = 0;
    CUtensorMap map_x16_16{}, map_x16_64{}, map_xp16{}, map_xp64{}, map_ep16{}, map_ep64{};
    // decode path (batch <= kDecMaxBatch): route+scatter -> fused expert GEMM -> combine
    DBuf vcodes, vscale, q_tier, q_first, e_q, scaling_d;            // rank-r projection tables
    DBuf dec_xperm, dec_extperm, dec_yslot, dec_cnt, dec_inv, dec_zq, dec_scratch, dec_segcnt, dec_ticket;
    int64_t dec_atom_rows = 0;
    bool dec_ready = false;
    std::atomic<uint64_t> launches{0};
    // comparison layouts (infer.cpp:187-339): decoded factors kept on the host
    // (decode_block_i8, codec.cpp:122-129) and device copies built on demand
    struct {
        int64_t M = 0, N = 0, R = 0;
        std::vector<float> U, V, sigma, scaling;   // M x o x r, N x r x i, r, K x i
        std::vector<uint16_t> placement;           // K x 2 (p, q)
    } lay;
    DBuf lay_U, lay_right, lay_proj1d, lay_sigma, lay_dq;
    bool lay_ready[4] = {false, false, false, false};
    int num_sms = 148;
    bool vq = false;                    // codebook residuals, expanded to fp16 weight blocks at load
    bool dense = false;                 // residuals held as dense fp16 weight blocks (codebook / odd group size)
    int art_bits = 0;                   // residual code width as stored in the artifact
    int64_t art_gs = 0;                 // scale group size as stored in the artifact
    // expert-GEMM device timing (tq_gemm_timing_enable)
    bool timing = false;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> tev;
    // TQ_KTIME=1 (diagnostics): an event after every launch of a forward; the
    // gaps between consecutive events (device time per kernel, launch gaps
    // included) are accumulated and printed when the layer is freed
    bool ktime = getenv("TQ_KTIME") && atoi(getenv("TQ_KTIME")) == 1;
    std::vector<std::vector<cudaEvent_t>> kev;   // one group per forward
    cudaStream_t kt_stream = nullptr;
    bool kt_active = false;
    void ktime_report() {
        std::vector<double> sum;
        int64_t n = 0;
        for (auto& grp : kev) {
            if (grp.size() < 2) continue;
            cudaEventSynchronize(grp.back());
            if (sum.size() < grp.size() - 1) sum.resize(grp.size() - 1, 0.0);
            for (size_t t = 1; t < grp.size(); ++t) {
                float ms = 0.0f;
                cudaEventElapsedTime(&ms, grp[t - 1], grp[t]);
                sum[t - 1] += ms;
            }
            ++n;
        }
        for (size_t t = 0; t < sum.size() && n > 0; ++t)
            fprintf(stderr, "ktime launch %zu: %.2f us (mean of %lld forwards)\n", t, sum[t] / n * 1e3,
                    static_cast<long long>(n));
        for (auto& grp : kev)
            for (auto e : grp) cudaEventDestroy(e);
        kev.clear();
    }
    // CUDA graphs of whole forwards, keyed by their arguments: one launch per
    // forward instead of six, no host work between the kernels
    struct GraphEntry {
        const void* key[6];
        int64_t batch;
        int path;
        cudaGraphExec_t exec;
        uint64_t launches;
    };
    std::vector<GraphEntry> graphs;
    cudaStream_t cap_stream = nullptr;
    bool use_graphs = !(getenv("TQ_GRAPHS") && atoi(getenv("TQ_GRAPHS")) == 0) && !getenv("TQ_DEBUG");  // debug dumps sync
    void drop_graphs() {
        // an executable graph may still be running (forwards are asynchronous): wait
        // for the device before its exec and the buffers it references are released
        if (!graphs.empty()) cudaDeviceSynchronize();
        for (auto& g : graphs) cudaGraphExecDestroy(g.exec);
        graphs.clear();
    }
    ~tq_layer() {
        for (auto& e : tev) {
            cudaEventDestroy(e.first);
            cudaEventDestroy(e.second);
        }
        drop_graphs();
        if (cap_stream) cudaStreamDestroy(cap_stream);
        if (ktime) ktime_report();
    }
};

namespace {

int64_t round_up(int64_t a, int64_t b) { return (a + b - 1) / b * b; }

// activation / output rows of a forward: routed slots with every expert's rows
// padded to a multiple of 8 (tile starts 8-row aligned for the swizzled
// bulk-copy layout), the shared-expert rows, and slack for 16-row MMA tiles
int64_t rows_for(const tq_layer* L, int64_t batch) {
    return batch * L->g.top_k + 8 * L->g.K + L->g.S * batch + 32;
}
int64_t compact_rows(const tq_layer* L, int64_t batch) { return batch * L->g.top_k + L->g.S * batch; }

// Upper bound of the split-K count the plan kernel may choose for a batch
// (it picks the best-balanced value <= this from the actual routing).
int proj_nsplit(const tq_layer* L, int64_t batch) {
    if (L->proj_mb == 0) return 1;
    const int64_t base = L->proj_mb * ((batch + 191) / 192);
    int64_t ns = (L->num_sms + base - 1) / base;
    ns = std::min<int64_t>(ns, std::max<int64_t>(1, L->g.kc_total / 4));
    return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ns, 32)));
}

struct LaunchCfg {
    int kc;        // K elements per chunk (64 or 128)
    int dn;        // TMEM accumulator columns (max token tile)
    int bn;        // token tile
    int kc_total;  // chunks per weight row
    int n_ext;     // extension chunks
};

int gemm_dn_host(int kc) { return kc == 64 ? 192 : 128; }

// Decode-sized batches (few tokens per expert) use 128-wide chunks and 16
// dequant warps; prefill uses 64-wide chunks and 192-token tiles.
LaunchCfg cfg_for(const tq_layer* L, int64_t batch) {
    // Batches up to kDecMaxBatch tokens run the decode path (tq_decode.cu); the
    // grouped path below serves larger batches and the expert-parallel stages with
    // its 64-column-chunk, 192-token-tile configuration only (the kc = 128
    // "mid" / resident-activation configurations of round 1 were retired: their
    // multi-unit ring bookkeeping faulted intermittently)
    (void)batch;
    LaunchCfg c;
    c.kc = 64;
    c.dn = 192;
    c.bn = c.dn;
    c.kc_total = static_cast<int>(L->g.k_pad / c.kc);
    c.n_ext = static_cast<int>((L->g.G + L->g.r + c.kc - 1) / c.kc);
    return c;
}

LaunchCfg cfg64(const tq_layer* L);

// the expert pass's config for a path: the lotile-only pass (extension chunks
// only, no packed codes) runs on the activation-ring configuration -- its units
// are one chunk each, and the decode configurations' per-unit pipeline makes
// them slower there (measured 58 vs 95 us at B=1 on c2, tools/layouts_bench.py)
LaunchCfg main_cfg(const tq_layer* L, int64_t batch, int path) {
    if (path == TQ_PATH_LOTILE) return cfg64(L);
    return cfg_for(L, batch);
}

// projection pass: dense fp16 operand from the row-major x16 buffer -- never
// the resident-activation decode configuration
LaunchCfg proj_cfg(const tq_layer* L, int64_t batch) {
    LaunchCfg c = cfg_for(L, batch);
    if (c.dn == 32) {
        c.dn = 64;
        c.bn = 64;
    }
    return c;
}

// decode configuration (dn == 32): resident activation slots of kc-wide chunks
// must fit ~140 KB of shared memory -> lower bound on the split-K count
static int ns_force() { return 0; }   // (experiment hook retired: the plan picks the K split)

int xr_ns_min(const tq_layer* L, const LaunchCfg& cf, int64_t batch) {
    if (cf.dn != 32) return 1;
    if (ns_force() > 0) return static_cast<int>(std::min<int64_t>(ns_force(), std::max<int64_t>(1, cf.kc_total / 2)));
    const int64_t tok = std::max<int64_t>(1, std::min<int64_t>(cf.bn, batch * L->g.top_k));
    const int64_t rows = (tok + 15) / 16 * 16;
    const int64_t slot = (cf.kc / 64) * rows * 128;
    // small tiles (B <= 8 per expert): keep the resident slots to ~40 KB so the code
    // ring gets ~24 stages (>150 KB of HBM reads in flight per SM); the plan's split
    // choice (several K splits at this size anyway) honours the bound
    const int64_t budget = rows <= 16 ? 40 * 1024 : 140 * 1024;
    const int64_t max_slots = std::min<int64_t>(64, budget / slot);
    const int64_t main_slots = std::max<int64_t>(1, max_slots - cf.n_ext);
    return static_cast<int>((cf.kc_total + main_slots - 1) / main_slots);
}

int xr_slots(const LaunchCfg& cf, int ns_min) {
    return (cf.kc_total + ns_min - 1) / ns_min + cf.n_ext;
}

int main_nsplit(const tq_layer* L, int64_t batch) {
    const int64_t local = L->e_end - L->e_begin;
    const int64_t active = std::max<int64_t>(1, std::min<int64_t>(local, batch * L->g.top_k) + L->g.S);
    const int64_t base = active * L->g.mb_count;
    int64_t ns = (16 * L->num_sms + base - 1) / base;
    // >= 4 main chunks per unit on the decode path: 2-chunk units pay the per-unit
    // pipeline cost twice as often and measured slower (TQ_NS_FORCE=16)
    ns = std::min<int64_t>(ns, std::max<int64_t>(1, L->g.kc_total / (cfg_for(L, batch).dn == 32 ? 4 : 2)));
    ns = std::max<int64_t>(1, std::min<int64_t>(ns, 16));
    if (ns_force() > 0 && cfg_for(L, batch).dn == 32) return xr_ns_min(L, cfg_for(L, batch), batch);
    return static_cast<int>(std::max<int64_t>(ns, xr_ns_min(L, cfg_for(L, batch), batch)));
}

void build_maps(tq_layer* L) {
    const int64_t rows = rows_for(L, L->cap);
    L->map_x16_16 = make_map(L->x16.p, L->cap, L->g.k_pad, 16);
    L->map_x16_64 = make_map(L->x16.p, L->cap, L->g.k_pad, 64);
    L->map_xp16 = make_map(L->xperm.p, rows, L->g.k_pad, 16);
    L->map_xp64 = make_map(L->xperm.p, rows, L->g.k_pad, 64);
    L->map_ep16 = make_map(L->extperm.p, rows, L->g.ext_cols, 16);
    L->map_ep64 = make_map(L->extperm.p, rows, L->g.ext_cols, 64);
}

void reserve(tq_layer* L, int64_t max_tokens) {
    if (max_tokens <= L->cap) return;
    L->drop_graphs();
    cuda_check(cudaSetDevice(L->device), "cudaSetDevice");
    const Geometry& g = L->g;
    const int64_t cap = round_up(std::max<int64_t>(max_tokens, 16), 16);
    const int64_t rows = rows_for(L, cap);
    int64_t ymax = 0, zmax = 0;
    for (int64_t b = 1; b <= cap; b = (b < 256 ? b + 1 : b + 64)) {
        ymax = std::max<int64_t>(ymax, main_nsplit(L, b) * rows_for(L, b) * g.o);
        zmax = std::max<int64_t>(zmax, proj_nsplit(L, b) * b * std::max<int64_t>(1, L->proj_rows));
    }
    ymax = std::max<int64_t>(ymax, main_nsplit(L, cap) * rows * g.o);
    zmax = std::max<int64_t>(zmax, proj_nsplit(L, cap) * cap * std::max<int64_t>(1, L->proj_rows));
    L->ids.alloc(sizeof(int32_t) * cap * g.top_k);
    L->gates.alloc(sizeof(float) * cap * g.top_k);
    L->x16.alloc(sizeof(__half) * cap * g.k_pad);
    L->sx.alloc(sizeof(float) * cap * std::max<int64_t>(1, g.G));
    L->route_ws.alloc(sizeof(float) * cap * g.K);
    L->route_ticket.alloc(sizeof(int32_t) * cap);
    cuda_check(cudaMemset(L->route_ticket.p, 0, sizeof(int32_t) * cap), "cudaMemset");
    L->perm.alloc(sizeof(int32_t) * cap * g.top_k);
    L->inv.alloc(sizeof(int32_t) * cap * g.top_k);
    L->offsets.alloc(sizeof(int32_t) * (g.K + 1));
    L->poffsets.alloc(sizeof(int32_t) * (g.K + 1));
    const int64_t max_units = (g.K + g.S) * g.mb_count * ((cap + 127) / 128 + g.K) * 16 + 64;
    L->units.alloc(sizeof(Unit) * max_units);
    L->n_units.alloc(sizeof(int32_t));
    L->nsplit_d.alloc(sizeof(int32_t));
    L->punits.alloc(sizeof(Unit) * (std::max<int64_t>(1, L->proj_mb) * ((cap + 127) / 128) * 32 + 8));
    L->n_punits.alloc(sizeof(int32_t));
    L->zpart.alloc(sizeof(float) * zmax);
    L->xperm.alloc(sizeof(__half) * rows * g.k_pad);
    L->extperm.alloc(sizeof(__half) * rows * g.ext_cols);
    L->ypart.alloc(sizeof(float) * ymax);
    L->xin.alloc(sizeof(float) * cap * g.i);
    L->yout.alloc(sizeof(float) * cap * g.o);
    cuda_check(cudaMemset(L->offsets.p, 0, sizeof(int32_t) * (g.K + 1)), "cudaMemset");
    if (!L->err_flag.p) {
        L->err_flag.alloc(sizeof(int32_t));
        cuda_check(cudaMemset(L->err_flag.p, 0, sizeof(int32_t)), "cudaMemset");
    }
    L->ypart_cap_floats = ymax;
    L->zpart_cap_floats = zmax;
    L->cap = cap;
    build_maps(L);
}

// Host image of an artifact: every tensor read and validated, nothing on the
// device yet (the reference's LoadedArtifact::layer, io.hpp:47-53, in wire form).
struct HostArtifact {
    int64_t K = 0, top_k = 0, i = 0, o = 0, S = 0, M = 0, N = 0, r = 0;
    std::vector<uint8_t> gate_b;        // K x i f32 (raw bytes)
    std::vector<float> scaling;         // K x i
    std::vector<uint16_t> placement;    // K x 2 (p, q)
    std::vector<float> sigma;           // r decoded singulars
    std::vector<uint8_t> u_b, v_b;      // int8 factor codes M x o x r, N x r x i
    std::vector<float> uabs, vabs;      // M, N
    std::vector<QMat> routed, shared;   // K, S residuals
};

// Geometry / placement checks every source shares (lotile_forward's
// FormatError for an out-of-grid cell, infer.cpp:61-72; layer spec checks of
// read_artifact, io.cpp:700-712).
void check_host_artifact(const HostArtifact& a) {
    if (a.K < 1) fail(TQ_ERR_FORMAT, "manifest spec invalid: layer spec: num_experts must be >= 1");
    if (a.top_k < 1 || a.top_k > a.K)
        fail(TQ_ERR_FORMAT, "manifest spec invalid: layer spec: top_k " + std::to_string(a.top_k) + " outside [1, " +
                                std::to_string(a.K) + "]");
    if (a.i < 1 || a.o < 1) fail(TQ_ERR_FORMAT, "manifest spec invalid: layer spec: dims must be >= 1");
    if (a.M == 0 || a.N == 0 || a.r == 0) fail(TQ_ERR_FORMAT, "manifest tiling meta: grid and rank must be nonzero");
    for (int64_t e = 0; e < a.K; ++e)
        if (a.placement[2 * e] >= a.M || a.placement[2 * e + 1] >= a.N)
            fail(TQ_ERR_FORMAT, "tensor 'placement': cell outside the tile grid");
    if (static_cast<int64_t>(a.routed.size()) != a.K || static_cast<int64_t>(a.shared.size()) != a.S)
        fail(TQ_ERR_FORMAT, "layer holds " + std::to_string(a.routed.size()) + " routed / " +
                                std::to_string(a.shared.size()) + " shared residuals, spec says " +
                                std::to_string(a.K) + " / " + std::to_string(a.S));
}

// read_artifact (io.cpp:679-813): manifest, every tensor's dtype / shape /
// byte_length / CRC32, placement bounds / injectivity / L1, residuals.  The
// residual blobs (all but ~2 MB of an artifact) are read, CRC-checked and
// unpacked by a pool of host threads, one matrix per task.
HostArtifact read_artifact_dir(const std::string& dir, bool verify) {
    Container c(dir, verify);
    const json& meta = c.meta();
    const json& s = require_object(meta, "spec");
    HostArtifact a;
    a.K = static_cast<int64_t>(require_size(s, "num_experts"));
    a.top_k = static_cast<int64_t>(require_size(s, "top_k"));
    a.i = static_cast<int64_t>(require_size(s, "in_dim"));
    a.o = static_cast<int64_t>(require_size(s, "out_dim"));
    a.S = static_cast<int64_t>(require_size(s, "num_shared"));
    if (a.K < 1) fail(TQ_ERR_FORMAT, "manifest spec invalid: layer spec: num_experts must be >= 1");
    if (a.top_k < 1 || a.top_k > a.K)
        fail(TQ_ERR_FORMAT, "manifest spec invalid: layer spec: top_k " + std::to_string(a.top_k) + " outside [1, " +
                                std::to_string(a.K) + "]");
    if (a.i < 1 || a.o < 1) fail(TQ_ERR_FORMAT, "manifest spec invalid: layer spec: dims must be >= 1");
    const json& tiling = require_object(meta, "tiling");
    a.M = static_cast<int64_t>(require_size(tiling, "grid_rows"));
    a.N = static_cast<int64_t>(require_size(tiling, "grid_cols"));
    a.r = static_cast<int64_t>(require_size(tiling, "rank"));
    if (a.M == 0 || a.N == 0 || a.r == 0) fail(TQ_ERR_FORMAT, "manifest tiling meta: grid and rank must be nonzero");

    const size_t K = static_cast<size_t>(a.K), I = static_cast<size_t>(a.i), O = static_cast<size_t>(a.o);
    const size_t M = static_cast<size_t>(a.M), N = static_cast<size_t>(a.N), R = static_cast<size_t>(a.r);
    std::vector<size_t> shape;
    a.gate_b = c.bytes("gate_weights", "f32", &shape);
    if (shape != std::vector<size_t>{K, I})
        fail(TQ_ERR_FORMAT, "tensor 'gate_weights': expected shape [" + std::to_string(K) + ", " + std::to_string(I) + "]");
    std::vector<uint8_t> scaling_b = c.bytes("scaling", "f32", &shape);
    if (shape != std::vector<size_t>{K, I})
        fail(TQ_ERR_FORMAT, "tensor 'scaling': expected shape [" + std::to_string(K) + ", " + std::to_string(I) + "]");
    a.scaling.resize(K * I);
    std::memcpy(a.scaling.data(), scaling_b.data(), scaling_b.size());
    // placement (io.cpp:731-760)
    const size_t l1 = require_size(tiling, "total_l1_displacement");
    if (!tiling.contains("ideal") || !tiling["ideal"].is_array() || tiling["ideal"].size() != K)
        fail(TQ_ERR_FORMAT, "manifest tiling meta: ideal must list every expert's cell");
    std::vector<std::pair<size_t, size_t>> ideal(K);
    for (size_t e = 0; e < K; ++e) {
        const json& cell = tiling["ideal"][e];
        if (!cell.is_array() || cell.size() != 2 || !cell[0].is_number_unsigned() || !cell[1].is_number_unsigned())
            fail(TQ_ERR_FORMAT, "manifest tiling meta: malformed ideal cell");
        ideal[e] = {cell[0].get<size_t>(), cell[1].get<size_t>()};
    }
    std::vector<uint8_t> pl_b = c.bytes("placement", "u16", &shape);
    if (shape != std::vector<size_t>{K, 2})
        fail(TQ_ERR_FORMAT, "tensor 'placement': expected shape [" + std::to_string(K) + ", 2]");
    a.placement.resize(K * 2);
    std::memcpy(a.placement.data(), pl_b.data(), pl_b.size());
    {
        std::set<std::pair<size_t, size_t>> seen;
        size_t dist = 0;
        for (size_t e = 0; e < K; ++e) {
            const std::pair<size_t, size_t> cell{a.placement[2 * e], a.placement[2 * e + 1]};
            if (cell.first >= M || cell.second >= N) fail(TQ_ERR_FORMAT, "tensor 'placement': cell outside the tile grid");
            if (!seen.insert(cell).second)
                fail(TQ_ERR_FORMAT, "tensor 'placement': duplicate cell (placement must be injective)");
            const size_t dr = cell.first > ideal[e].first ? cell.first - ideal[e].first : ideal[e].first - cell.first;
            const size_t dc = cell.second > ideal[e].second ? cell.second - ideal[e].second : ideal[e].second - cell.second;
            dist += dr + dc;
        }
        if (dist != l1)
            fail(TQ_ERR_FORMAT, "manifest tiling meta: total_l1_displacement does not match the stored cells");
    }
    // factors
    std::vector<uint8_t> sing_b = c.bytes("tiled.singulars", "f16-roundtrip", &shape);
    if (shape != std::vector<size_t>{R}) fail(TQ_ERR_FORMAT, "tensor 'tiled.singulars': unexpected shape");
    a.sigma.resize(R);
    for (size_t j = 0; j < R; ++j) {
        uint16_t hb;
        std::memcpy(&hb, sing_b.data() + 2 * j, 2);
        a.sigma[j] = half_bits_to_float(hb);
    }
    a.u_b = c.bytes("tiled.u.codes", "u8", &shape);
    if (shape != std::vector<size_t>{M, O, R}) fail(TQ_ERR_FORMAT, "tensor 'tiled.u.codes': unexpected shape");
    std::vector<uint8_t> uabs_b = c.bytes("tiled.u.absmax", "f32", &shape);
    if (shape != std::vector<size_t>{M}) fail(TQ_ERR_FORMAT, "tensor 'tiled.u.absmax': expected shape [" + std::to_string(M) + "]");
    a.v_b = c.bytes("tiled.v.codes", "u8", &shape);
    if (shape != std::vector<size_t>{N, R, I}) fail(TQ_ERR_FORMAT, "tensor 'tiled.v.codes': unexpected shape");
    std::vector<uint8_t> vabs_b = c.bytes("tiled.v.absmax", "f32", &shape);
    if (shape != std::vector<size_t>{N}) fail(TQ_ERR_FORMAT, "tensor 'tiled.v.absmax': expected shape [" + std::to_string(N) + "]");
    a.uabs.resize(M);
    a.vabs.resize(N);
    std::memcpy(a.uabs.data(), uabs_b.data(), uabs_b.size());
    std::memcpy(a.vabs.data(), vabs_b.data(), vabs_b.size());

    // residuals: K routed + S shared matrices, read in parallel; the first
    // failing matrix in (routed, shared) order is reported, as a serial reader would
    const json& qmeta = require_object(meta, "quant");
    const json* smeta = a.S > 0 ? &require_object(meta, "shared_quant") : nullptr;
    const size_t total = K + static_cast<size_t>(a.S);
    std::vector<QMat> mats(total);
    std::vector<std::exception_ptr> errs(total);
    {
        std::atomic<size_t> next{0};
        auto work = [&] {
            for (size_t w = next++; w < total; w = next++) {
                try {
                    if (w < K) mats[w] = read_qmat(c, "expert." + std::to_string(w), qmeta, O, I);
                    else mats[w] = read_qmat(c, "sharedexpert." + std::to_string(w - K), *smeta, O, I);
                } catch (...) {
                    errs[w] = std::current_exception();
                }
            }
        };
        const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
        std::vector<std::thread> pool;
        for (unsigned t = 1; t < std::min<unsigned>(hw, static_cast<unsigned>(total)); ++t) pool.emplace_back(work);
        work();
        for (auto& t : pool) t.join();
    }
    for (size_t w = 0; w < total; ++w)
        if (errs[w]) std::rethrow_exception(errs[w]);
    a.routed.assign(std::make_move_iterator(mats.begin()), std::make_move_iterator(mats.begin() + K));
    a.shared.assign(std::make_move_iterator(mats.begin() + K), std::make_move_iterator(mats.end()));
    return a;
}

// In-memory layer (TileQLayer, infer.hpp:22-28) through the C-ABI descriptor:
// the same checks the reader applies to the same fields (io.cpp:422-485 for
// residuals) minus those that only exist on the wire (CRC, byte lengths).
HostArtifact artifact_from_desc(const tq_layer_desc* d) {
    if (!d) fail(TQ_ERR_PARAM, "tq_layer_create: null descriptor");
    HostArtifact a;
    a.K = d->num_experts;
    a.top_k = d->top_k;
    a.i = d->in_dim;
    a.o = d->out_dim;
    a.S = d->num_shared;
    a.M = d->grid_rows;
    a.N = d->grid_cols;
    a.r = d->rank;
    if (a.K < 1 || a.i < 1 || a.o < 1 || a.S < 0 || a.M < 0 || a.N < 0 || a.r < 0)
        fail(TQ_ERR_SHAPE, "tq_layer_create: layer dimensions must be positive");
    if (a.top_k < 1 || a.top_k > a.K)
        fail(TQ_ERR_PARAM, "tq_layer_create: top_k " + std::to_string(a.top_k) + " outside [1, " + std::to_string(a.K) + "]");
    const size_t K = static_cast<size_t>(a.K), I = static_cast<size_t>(a.i), O = static_cast<size_t>(a.o);
    const size_t M = static_cast<size_t>(a.M), N = static_cast<size_t>(a.N), R = static_cast<size_t>(a.r);
    if (!d->gate_weights || !d->scaling || !d->placement || !d->singular_bits || !d->u_codes || !d->u_absmax ||
        !d->v_codes || !d->v_absmax || !d->experts || (a.S > 0 && !d->shared))
        fail(TQ_ERR_PARAM, "tq_layer_create: null tensor pointer in the descriptor");
    a.gate_b.resize(K * I * 4);
    std::memcpy(a.gate_b.data(), d->gate_weights, a.gate_b.size());
    a.scaling.assign(d->scaling, d->scaling + K * I);
    for (float v : a.scaling)
        if (!(v > 0.0f) || !std::isfinite(v)) fail(TQ_ERR_FORMAT, "tensor 'scaling': entries must be positive and finite");
    a.placement.resize(K * 2);
    for (size_t t = 0; t < K * 2; ++t) {
        if (d->placement[t] > 0xFFFFu) fail(TQ_ERR_FORMAT, "tensor 'placement': cell outside the tile grid");
        a.placement[t] = static_cast<uint16_t>(d->placement[t]);
    }
    a.sigma.resize(R);
    for (size_t j = 0; j < R; ++j) a.sigma[j] = half_bits_to_float(d->singular_bits[j]);
    a.u_b.assign(reinterpret_cast<const uint8_t*>(d->u_codes), reinterpret_cast<const uint8_t*>(d->u_codes) + M * O * R);
    a.v_b.assign(reinterpret_cast<const uint8_t*>(d->v_codes), reinterpret_cast<const uint8_t*>(d->v_codes) + N * R * I);
    a.uabs.assign(d->u_absmax, d->u_absmax + M);
    a.vabs.assign(d->v_absmax, d->v_absmax + N);
    auto qm = [&](const tq_qmat_desc& q, const std::string& name) {
        QMat m;
        m.bits = q.bits;
        if (q.bits != 2 && q.bits != 3 && q.bits != 4 && q.bits != 8)
            fail(TQ_ERR_PARAM, "tensor '" + name + "': bits must be one of 2, 3, 4, 8");
        m.vec = q.mode == TQ_QUANT_VECTOR;
        if (!m.vec && q.mode != TQ_QUANT_SCALAR) fail(TQ_ERR_PARAM, "tensor '" + name + "': unknown quant mode");
        if (static_cast<size_t>(q.out_dim) != O || static_cast<size_t>(q.in_dim) != I)
            fail(TQ_ERR_SHAPE, "tensor '" + name + "': residual is " + std::to_string(q.out_dim) + "x" +
                                   std::to_string(q.in_dim) + ", layer is " + std::to_string(O) + "x" + std::to_string(I));
        size_t count;
        if (!m.vec) {
            if (q.group_size < 1) fail(TQ_ERR_PARAM, "tensor '" + name + "': group_size must be >= 1");
            m.gs = static_cast<size_t>(q.group_size);
            const size_t G = (I + m.gs - 1) / m.gs;
            count = O * I;
            if (!q.scale_bits || !q.zeros) fail(TQ_ERR_PARAM, "tensor '" + name + "': null scale/zero table");
            m.scales.assign(q.scale_bits, q.scale_bits + O * G);
            m.zeros.assign(q.zeros, q.zeros + O * G);
            for (size_t t = 0; t < m.scales.size(); ++t) {
                const float sv = half_bits_to_float(m.scales[t]);
                if (!(sv > 0.0f) || !std::isfinite(sv)) fail(TQ_ERR_FORMAT, "tensor '" + name + ".scales': non-positive scale");
                if (m.zeros[t] >> q.bits) fail(TQ_ERR_FORMAT, "tensor '" + name + ".zeros': zero point outside [0, 2^bits)");
            }
        } else {
            if (q.sub_dim < 1) fail(TQ_ERR_PARAM, "tensor '" + name + "': sub_dim must be >= 1");
            m.sub_dim = static_cast<size_t>(q.sub_dim);
            count = O * ((I + m.sub_dim - 1) / m.sub_dim);
            if (!q.codebook_bits) fail(TQ_ERR_PARAM, "tensor '" + name + "': null codebook");
            m.codebook.assign(q.codebook_bits, q.codebook_bits + (size_t{1} << q.bits) * m.sub_dim);
        }
        if (!q.packed || static_cast<size_t>(q.packed_bytes) != packed_byte_length(count, q.bits))
            fail(TQ_ERR_SIZE, "tensor '" + name + ".codes': packed stream holds " + std::to_string(q.packed_bytes) +
                                  " bytes, expected " + std::to_string(packed_byte_length(count, q.bits)));
        m.packed.assign(q.packed, q.packed + q.packed_bytes);
        return m;
    };
    for (size_t e = 0; e < K; ++e) a.routed.push_back(qm(d->experts[e], "expert." + std::to_string(e)));
    for (int64_t s2 = 0; s2 < a.S; ++s2) a.shared.push_back(qm(d->shared[s2], "sharedexpert." + std::to_string(s2)));
    check_host_artifact(a);
    return a;
}

// Engine layout from a validated host image; device work starts only once
// every host-side check has passed.
void build_layer(tq_layer* L, HostArtifact& a, int device, int64_t e_begin, int64_t e_end) {
    check_host_artifact(a);
    Geometry& g = L->g;
    g.K = a.K;
    g.top_k = a.top_k;
    g.i = a.i;
    g.o = a.o;
    g.S = a.S;
    g.M = a.M;
    g.N = a.N;
    g.r = a.r;
    const size_t K = static_cast<size_t>(g.K), I = static_cast<size_t>(g.i), O = static_cast<size_t>(g.o);
    const size_t M = static_cast<size_t>(g.M), N = static_cast<size_t>(g.N), R = static_cast<size_t>(g.r);
    const std::vector<uint8_t>& gate_b = a.gate_b;
    const std::vector<float>& scaling = a.scaling;
    const std::vector<uint16_t>& placement = a.placement;
    const std::vector<float>& sigma = a.sigma;
    const std::vector<uint8_t>& u_b = a.u_b;
    const std::vector<uint8_t>& v_b = a.v_b;
    const std::vector<float>& uabs = a.uabs;
    const std::vector<float>& vabs = a.vabs;
    {
        // host copies for the comparison layouts: value = float(code) * (absmax / 127.0f)
        L->lay.M = static_cast<int64_t>(M);
        L->lay.N = static_cast<int64_t>(N);
        L->lay.R = static_cast<int64_t>(R);
        L->lay.U.resize(M * O * R);
        for (size_t pb = 0; pb < M; ++pb) {
            const float sc = uabs[pb] / 127.0f;
            for (size_t t = 0; t < O * R; ++t)
                L->lay.U[pb * O * R + t] = static_cast<float>(static_cast<int8_t>(u_b[pb * O * R + t])) * sc;
        }
        L->lay.V.resize(N * R * I);
        for (size_t qb = 0; qb < N; ++qb) {
            const float sc = vabs[qb] / 127.0f;
            for (size_t t = 0; t < R * I; ++t)
                L->lay.V[qb * R * I + t] = static_cast<float>(static_cast<int8_t>(v_b[qb * R * I + t])) * sc;
        }
        L->lay.sigma = sigma;
        L->lay.scaling = scaling;
        L->lay.placement = placement;
    }

    // residual experts
    if (e_end < 0 || e_end > g.K) e_end = g.K;
    if (e_begin < 0 || e_begin > e_end) fail(TQ_ERR_PARAM, "expert range [" + std::to_string(e_begin) + ", " + std::to_string(e_end) + ") outside [0, K]");
    L->e_begin = e_begin;
    L->e_end = e_end;
    // prescale exponent of EVERY routed expert: a rank's dispatch rows carry
    // the low-rank term pre-multiplied by the owner's 2^k (expert parallel)
    std::vector<int> k_all(K, 0);
    for (size_t e = 0; e < K; ++e) k_all[e] = prescale_exponent(a.routed[e]);
    const QMat& q0 = a.routed[0];
    for (size_t w = 1; w < K; ++w)
        if (a.routed[w].bits != q0.bits || a.routed[w].vec != q0.vec || a.routed[w].gs != q0.gs ||
            a.routed[w].sub_dim != q0.sub_dim)
            fail(TQ_ERR_PARAM, "routed experts must share one bits/mode/group_size on the GPU engine");
    for (const QMat& m : a.shared)
        if (m.bits != q0.bits || m.vec != q0.vec || m.gs != q0.gs || m.sub_dim != q0.sub_dim)
            fail(TQ_ERR_PARAM, "shared experts must use the routed experts' bits/group_size on the GPU engine");
    // codebook (vector) residuals, quant.cpp:303-321: every codebook entry is f16-snapped
    // (quant.cpp:262-266), so the dequantized weights ARE fp16 values -- the loader
    // resolves each code through its expert's codebook into exact fp16 weight blocks,
    // streamed by the dense (kDenseBits) weight path; unit scales, no zero points
    const bool vq = q0.vec;
    // scale groups that are not a multiple of 32 codes (the dequant works on 32-code
    // super-words per scale): the loader dequantizes such residuals once, exactly in
    // f64 and rounded once to fp16 (prescaled by 2^k like the code path), into dense
    // weight blocks -- the same dense-weight path as codebook residuals
    const bool dense_scalar = !vq && q0.gs % 32 != 0;
    L->vq = vq;
    L->dense = vq || dense_scalar;
    L->art_bits = q0.bits;
    L->art_gs = static_cast<int64_t>(q0.gs);
    const int bits = L->dense ? kDenseBits : q0.bits;
    const size_t gs = L->dense ? 128 : q0.gs;
    std::vector<QMat> q;
    for (int64_t e = e_begin; e < e_end; ++e) q.push_back(std::move(a.routed[static_cast<size_t>(e)]));
    for (auto& m : a.shared) q.push_back(std::move(m));
    g.bits = bits;
    g.gs = static_cast<int64_t>(gs);
    if (g.gs % 32 != 0)
        fail(TQ_ERR_PARAM, "group_size " + std::to_string(g.gs) +
                               " is not a multiple of 32; the GPU engine dequantizes 32-code super-words per group");
    g.G = (g.i + g.gs - 1) / g.gs;
    g.k_pad = round_up(g.i, kKC);
    g.kc_total = g.k_pad / kKC;
    g.o_pad = round_up(g.o, kBM);
    g.mb_count = g.o_pad / kBM;
    g.n_ext = (g.G + g.r + kKC - 1) / kKC;   // extension chunks at KC = 64
    g.ext_cols = round_up(g.G + g.r, 256);    // room for KC = 256 chunks (zero-padded)
    if (g.K > 64)
        fail(TQ_ERR_PARAM, "GPU engine routes at most 64 experts (num_experts " + std::to_string(g.K) + ")");
    if (g.G > 64 || g.r > 64)
        fail(TQ_ERR_PARAM, "GPU engine supports at most 64 scale groups per row and rank <= 64 (groups " +
                               std::to_string(g.G) + ", rank " + std::to_string(g.r) + ")");
    L->n_weights = static_cast<int64_t>(q.size());

    // --- repack residuals (parallel over matrices) ---
    const int64_t blk = code_block_bytes(bits);
    L->weight_stride = g.mb_count * g.kc_total * blk;
    const int64_t slab = g.mb_count * g.G * kBM;  // scale / zero entries per matrix
    // scalar code streams are repacked on the device after upload (below); only the
    // dense-weight paths (codebook / odd group sizes) build their blocks on the host
    const bool device_repack = !L->dense;
    std::vector<uint8_t> h_codes(device_repack ? 0 : static_cast<size_t>(L->weight_stride * L->n_weights));
    std::vector<uint16_t> h_scales(static_cast<size_t>(slab * L->n_weights));
    std::vector<uint8_t> h_zeros(static_cast<size_t>(slab * L->n_weights));
    std::vector<int> wk(static_cast<size_t>(L->n_weights), 0);
    {
        std::vector<std::thread> pool;
        std::vector<std::string> errs(q.size());
        const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
        std::atomic<size_t> next{0};
        for (unsigned t = 0; t < std::min<unsigned>(hw, static_cast<unsigned>(q.size())); ++t)
            pool.emplace_back([&] {
                for (size_t w = next++; w < q.size(); w = next++) {
                    try {
                        if (vq)
                            repack_vq(q[w], g, h_codes.data() + w * L->weight_stride, h_scales.data() + w * slab,
                                      h_zeros.data() + w * slab, &wk[w]);
                        else if (dense_scalar)
                            repack_dense_scalar(q[w], g, h_codes.data() + w * L->weight_stride,
                                                h_scales.data() + w * slab, h_zeros.data() + w * slab, &wk[w]);
                        else
                            repack_slabs(q[w], g, h_scales.data() + w * slab, h_zeros.data() + w * slab, &wk[w]);
                    } catch (const std::exception& e) {
                        errs[w] = e.what();
                    }
                }
            });
        for (auto& t : pool) t.join();
        for (size_t w = 0; w < errs.size(); ++w)
            if (!errs[w].empty()) fail(TQ_ERR_FORMAT, errs[w]);
    }
    std::vector<std::vector<uint8_t>> packed_streams;
    if (device_repack)
        for (auto& m : q) packed_streams.push_back(std::move(m.packed));
    q.clear();
    std::vector<float> h_outscale(static_cast<size_t>(L->n_weights));
    for (int64_t w = 0; w < L->n_weights; ++w) h_outscale[w] = static_cast<float>(std::ldexp(1.0, -wk[w]));
    // Extension blocks per (weight, m-block): dense fp16 A-operand columns appended
    // after the main K range: [-zero * s' per scale group | U_p codes | 0].  They
    // depend only on (weight, row), so they are formed once here (-zero*s' rounded
    // once to fp16 like the device HMUL would; int8 U codes are exact in fp16).
    const int64_t n_ext64 = g.n_ext;
    const int eblk = code_block_bytes(kDenseBits);
    std::vector<uint8_t> h_ext(static_cast<size_t>(L->n_weights * g.mb_count * n_ext64 * eblk), 0);
    for (int64_t w = 0; w < L->n_weights; ++w) {
        const bool routed = w < e_end - e_begin;
        const size_t p_blk = routed ? placement[2 * (e_begin + w)] : 0;
        for (int64_t mb = 0; mb < g.mb_count; ++mb) {
            uint8_t* base = h_ext.data() + ((w * g.mb_count + mb) * n_ext64) * eblk;
            for (int64_t blk = 0; blk < n_ext64; ++blk) {
                uint16_t* b16 = reinterpret_cast<uint16_t*>(base + blk * eblk);
                for (int rl = 0; rl < kBM; ++rl) {
                    const int64_t row = mb * kBM + rl;
                    for (int col = 0; col < 64; ++col) {
                        const int64_t gc = blk * 64 + col;
                        float val = 0.0f;
                        if (row < g.o && gc < g.G) {
                            const size_t si = static_cast<size_t>(w * slab + (mb * g.G + gc) * kBM + rl);
                            const float sv = half_bits_to_float(h_scales[si]);
                            val = static_cast<float>(-static_cast<double>(h_zeros[si]) * sv);
                        } else if (row < g.o && routed && gc >= g.G && gc < g.G + g.r) {
                            val = static_cast<float>(static_cast<int8_t>(u_b[(p_blk * O + static_cast<size_t>(row)) * R +
                                                                              static_cast<size_t>(gc - g.G)]));
                        }
                        // block layout: u32 word (hh*16 + j) of row rl holds columns 32*hh + 2j (+1)
                        const int hh = col >> 5, j = (col & 31) >> 1, hi = col & 1;
                        b16[((hh * 16 + j) * kBM + rl) * 2 + hi] = float_to_half_bits(val);
                    }
                }
            }
        }
    }

    // --- descale tiers + projection matrices (infer.cpp:74-117) ---
    std::vector<int> tier(N, 0);
    std::vector<int64_t> first(N, -1);
    for (size_t qq = 0; qq < N; ++qq) {
        bool any = false, all_same = true, all_scalar = true;
        for (size_t k = 0; k < K; ++k) {
            if (placement[2 * k + 1] != qq) continue;
            const float* sk = &scaling[k * I];
            if (!any) {
                first[qq] = static_cast<int64_t>(k);
                any = true;
            } else if (!std::equal(sk, sk + I, &scaling[static_cast<size_t>(first[qq]) * I])) {
                all_same = false;
            }
            for (size_t cc = 0; cc < I; ++cc)
                if (sk[cc] != sk[0]) {
                    all_scalar = false;
                    break;
                }
        }
        tier[qq] = (!any || all_same) ? 0 : (all_scalar ? 1 : 2);
        L->tiers[tier[qq]]++;
    }
    // v values exactly as decode_block_i8 (codec.cpp:122-129)
    auto vval = [&](size_t qq, size_t j, size_t cc) {
        const float sc = vabs[qq] == 0.0f ? 0.0f : vabs[qq] / 127.0f;
        return static_cast<float>(static_cast<int8_t>(v_b[(qq * R + j) * I + cc])) * sc;
    };
    std::vector<std::vector<double>> mats;   // each r x i (double before fp16 rounding)
    std::vector<int32_t> pm_of(K, 0);
    std::vector<float> zscale(K, 1.0f);
    std::vector<int64_t> q_matrix(N, -1);
    for (size_t qq = 0; qq < N; ++qq) {
        if (tier[qq] == 2) continue;
        if (first[qq] < 0) continue;  // unused column block
        std::vector<double> m(R * I);
        for (size_t j = 0; j < R; ++j)
            for (size_t cc = 0; cc < I; ++cc) {
                double val = static_cast<double>(sigma[j]) * static_cast<double>(vval(qq, j, cc));
                if (tier[qq] == 0) val /= scaling[static_cast<size_t>(first[qq]) * I + cc];
                m[j * I + cc] = static_cast<double>(static_cast<float>(val));
            }
        q_matrix[qq] = static_cast<int64_t>(mats.size());
        mats.push_back(std::move(m));
    }
    for (size_t e = 0; e < K; ++e) {
        const size_t p = placement[2 * e], qq = placement[2 * e + 1];
        const float su = uabs[p] == 0.0f ? 0.0f : uabs[p] / 127.0f;
        double inv = 1.0;
        if (tier[qq] == 2) {
            std::vector<double> m(R * I);
            for (size_t j = 0; j < R; ++j)
                for (size_t cc = 0; cc < I; ++cc) {
                    const float prow = static_cast<float>(static_cast<double>(sigma[j]) * vval(qq, j, cc));
                    m[j * I + cc] = static_cast<double>(prow) / scaling[e * I + cc];
                }
            pm_of[e] = static_cast<int32_t>(mats.size());
            mats.push_back(std::move(m));
        } else {
            pm_of[e] = static_cast<int32_t>(q_matrix[qq]);
            if (tier[qq] == 1) inv = 1.0 / scaling[e * I];
        }
        const int k = k_all[e];
        zscale[e] = static_cast<float>(static_cast<double>(su) * inv * std::ldexp(1.0, k));
    }
    L->NP = static_cast<int64_t>(mats.size());
    L->proj_rows = L->NP * g.r;
    L->proj_o_pad = round_up(std::max<int64_t>(L->proj_rows, 1), kBM);
    L->proj_mb = L->proj_rows > 0 ? L->proj_o_pad / kBM : 0;
    // dense fp16 blocks of the stacked projection with per-row power-of-two normalisation
    const int dblk = code_block_bytes(kDenseBits);
    L->pweight_stride = L->proj_mb * g.kc_total * dblk;
    std::vector<uint8_t> h_p(static_cast<size_t>(std::max<int64_t>(L->pweight_stride, 16)), 0);
    std::vector<float> rowscale(static_cast<size_t>(std::max<int64_t>(L->proj_rows, 1)), 1.0f);
    std::vector<uint16_t> prow_h(I);
    for (int64_t pr = 0; pr < L->proj_rows; ++pr) {
        const std::vector<double>& m = mats[static_cast<size_t>(pr / g.r)];
        const size_t j = static_cast<size_t>(pr % g.r);
        double mx = 0.0;
        for (size_t cc = 0; cc < I; ++cc) mx = std::max(mx, std::fabs(m[j * I + cc]));
        int k = 0;
        if (mx > 0.0) k = static_cast<int>(std::floor(std::log2(mx))) - 9;
        rowscale[static_cast<size_t>(pr)] = static_cast<float>(std::ldexp(1.0, k));
        for (size_t cc = 0; cc < I; ++cc) prow_h[cc] = float_to_half_bits(static_cast<float>(std::ldexp(m[j * I + cc], -k)));
        const int64_t mb = pr / kBM, rl = pr % kBM;
        for (int64_t kc = 0; kc < g.kc_total; ++kc) {
            uint32_t* block = reinterpret_cast<uint32_t*>(h_p.data() + (mb * g.kc_total + kc) * dblk);
            for (int h = 0; h < 2; ++h)
                for (int jw = 0; jw < 16; ++jw) {
                    const int64_t c0 = kc * kKC + 32 * h + 2 * jw;
                    const uint32_t lo = c0 < g.i ? prow_h[static_cast<size_t>(c0)] : 0u;
                    const uint32_t hi = c0 + 1 < g.i ? prow_h[static_cast<size_t>(c0 + 1)] : 0u;
                    block[(h * 16 + jw) * kBM + rl] = lo | (hi << 16);
                }
        }
    }

    // --- device: only now that every host-side check has passed ---
    cuda_check(cudaSetDevice(device), "cudaSetDevice");
    L->device = device;
    {
        cudaDeviceProp prop;
        cuda_check(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
        if (prop.major != 10)
            fail(TQ_ERR_CUDA, "libtileq_b200 is built for sm_100a (B200); device " + std::to_string(device) +
                                  " is sm_" + std::to_string(prop.major) + std::to_string(prop.minor));
        L->num_sms = prop.multiProcessorCount;
    }
    // --- upload ---
    L->gate.upload(gate_b.data(), gate_b.size());
    if (device_repack) {
        // packed streams -> device -> engine blocks (repack_codes_kernel), one staging
        // buffer reused across matrices
        L->codes.alloc(static_cast<size_t>(L->weight_stride * L->n_weights));
        size_t max_stream = 0;
        for (const auto& ps : packed_streams) max_stream = std::max(max_stream, ps.size());
        DBuf staging;
        staging.alloc(max_stream);
        for (int64_t w = 0; w < L->n_weights; ++w) {
            const auto& ps = packed_streams[static_cast<size_t>(w)];
            cuda_check(cudaMemcpy(staging.p, ps.data(), ps.size(), cudaMemcpyHostToDevice), "packed stream H2D");
            cuda_check(launch_repack_codes(staging.as<uint8_t>(), static_cast<int64_t>(ps.size()), g.bits, g.o, g.i,
                                           g.mb_count, g.kc_total, L->codes.as<uint8_t>() + w * L->weight_stride,
                                           nullptr),
                       "repack launch");
        }
        cuda_check(cudaDeviceSynchronize(), "repack sync");   // staging is reused / freed
    } else {
        L->codes.upload(h_codes.data(), h_codes.size());
    }
    L->scales.upload(h_scales.data(), h_scales.size() * 2);
    L->ext_blocks.upload(h_ext.data(), h_ext.size());
    L->w_outscale.upload(h_outscale.data(), h_outscale.size() * 4);
    L->pcodes.upload(h_p.data(), h_p.size());
    const float one = 1.0f;
    L->p_outscale.upload(&one, 4);
    L->pm_of.upload(pm_of.data(), pm_of.size() * 4);
    L->zscale.upload(zscale.data(), zscale.size() * 4);
    L->rowscale.upload(rowscale.data(), rowscale.size() * 4);
    // decode path: rank-r projection tables -- the exact int8 V codes and the per-row
    // factor sigma_j * vabs_q / 127 (decode_block_i8, codec.cpp:122-129), the
    // descale tier of every tile column and the scaling vectors (infer.cpp:74-117)
    {
        std::vector<float> vsc(N * R);
        for (size_t qq = 0; qq < N; ++qq) {
            const float sc = vabs[qq] == 0.0f ? 0.0f : vabs[qq] / 127.0f;
            for (size_t j = 0; j < R; ++j)
                vsc[qq * R + j] = static_cast<float>(static_cast<double>(sigma[j]) * static_cast<double>(sc));
        }
        std::vector<int32_t> qt(N), qf(N), eq(K);
        for (size_t qq = 0; qq < N; ++qq) {
            qt[qq] = first[qq] < 0 ? -1 : tier[qq];
            qf[qq] = first[qq] < 0 ? 0 : static_cast<int32_t>(first[qq]);
        }
        for (size_t e = 0; e < K; ++e) eq[e] = placement[2 * e + 1];
        L->vcodes.upload(v_b.data(), v_b.size());
        L->vscale.upload(vsc.data(), vsc.size() * 4);
        L->q_tier.upload(qt.data(), qt.size() * 4);
        L->q_first.upload(qf.data(), qf.size() * 4);
        L->e_q.upload(eq.data(), eq.size() * 4);
        L->scaling_d.upload(scaling.data(), scaling.size() * 4);
    }
    L->device_bytes = static_cast<int64_t>(L->gate.n + L->codes.n + L->scales.n + L->ext_blocks.n + L->pcodes.n +
                                           L->rowscale.n);
    reserve(L, 64);
}

GemmParams base_params(tq_layer* L, const LaunchCfg& cf, int64_t max_tok) {
    GemmParams p;
    std::memset(&p, 0, sizeof(p));
    p.group_size = static_cast<int32_t>(L->g.gs);
    p.kc_total = cf.kc_total;
    p.kc_width = cf.kc;
    p.dn = cf.dn;
    p.n_ext_chunks = cf.n_ext;
    p.bn_max = static_cast<int32_t>(std::max<int64_t>(1, std::min<int64_t>(cf.bn, max_tok)));
    return p;
}

LaunchCfg cfg64(const tq_layer* L) {
    LaunchCfg c;
    c.kc = 64;
    c.dn = 192;
    c.bn = gemm_dn_host(64);
    c.kc_total = static_cast<int>(L->g.k_pad / 64);
    c.n_ext = static_cast<int>(L->g.n_ext);
    return c;
}

void count_launch(tq_layer* L, int n = 1) {
    L->launches += static_cast<uint64_t>(n);
#ifdef TQ_CHECK_EACH
    // diagnostics build: synchronize after every launch and name the failing one
    {
        const cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            fprintf(stderr, "TQ_CHECK_EACH: launch #%llu of the layer failed: %s\n",
                    static_cast<unsigned long long>(L->launches.load()), cudaGetErrorString(e));
            fail(TQ_ERR_CUDA, std::string("TQ_CHECK_EACH: ") + cudaGetErrorString(e));
        }
    }
#endif
    if (L->ktime && L->kt_active && !L->kev.empty()) {
        cudaEvent_t e;
        cudaEventCreate(&e);
        cudaEventRecord(e, L->kt_stream);
        L->kev.back().push_back(e);
    }
}

// prep (x16, sx) and optional routing (the plan runs as its own launch: fused into
// the router's last CTA it measured slower -- the plan's unit loop wants the full
// 1024-thread CTA)
void run_route(tq_layer* L, const float* x, int64_t batch, bool do_route, cudaStream_t st) {
    if (L->ktime) {
        L->kt_stream = st;
        L->kt_active = true;
        cudaEvent_t e;
        cudaEventCreate(&e);
        cudaEventRecord(e, st);
        L->kev.push_back({e});
    }
    cuda_check(launch_route(x, static_cast<int>(batch), static_cast<int>(L->g.i), L->gate.as<float>(),
                            do_route ? static_cast<int>(L->g.K) : 0, static_cast<int>(L->g.top_k),
                            static_cast<int>(L->g.gs), static_cast<int>(L->g.G), static_cast<int>(L->g.k_pad),
                            L->ids.as<int32_t>(), L->gates.as<float>(), L->x16.as<__half>(), L->sx.as<float>(),
                            L->route_ws.as<float>(), L->route_ticket.as<int32_t>(), st),
               "route_kernel launch");
    count_launch(L);
}

// The fused expert GEMM, bracketed by CUDA events on its own stream when the
// layer's timing hook is on (tq_gemm_timing_enable): the device time bench.py
// divides the kernel's algorithmic bytes / flops by.
static void timed_expert_gemm(tq_layer* L, const GemmParams& p, int grid, cudaStream_t st) {
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    if (L->timing) {
        cuda_check(cudaEventCreate(&ev0), "cudaEventCreate");
        cuda_check(cudaEventCreate(&ev1), "cudaEventCreate");
        cuda_check(cudaEventRecord(ev0, st), "cudaEventRecord");
    }
    cuda_check(launch_gemm(p, grid, st), "expert gemm launch");
    if (L->timing) {
        cuda_check(cudaEventRecord(ev1, st), "cudaEventRecord");
        L->tev.emplace_back(ev0, ev1);
    }
}

// the plan of one forward: permutation of `ids` and the GEMM work units
PlanArgs make_plan_args(tq_layer* L, int64_t batch, const int32_t* ids, int path) {
    const Geometry& g = L->g;
    const bool use_lotile = path != TQ_PATH_QMOE;
    const bool use_qmoe = path != TQ_PATH_LOTILE;
    const LaunchCfg cf = main_cfg(L, batch, path);
    const LaunchCfg cfp = proj_cfg(L, batch);
    const bool xr = cf.dn == 32;   // decode: resident activation tiles, contiguous unit runs
    const int ns_min = use_qmoe ? xr_ns_min(L, cf, batch) : 1;
    const int nsplit = use_qmoe ? main_nsplit(L, batch) : 1;
    const int pns = proj_nsplit(L, batch);
    const bool with_shared = use_qmoe && g.S > 0;
    PlanArgs pa{};
    pa.ids = ids;
    pa.batch = static_cast<int>(batch);
    pa.top_k = static_cast<int>(g.top_k);
    pa.num_experts = static_cast<int>(g.K);
    pa.e_begin = static_cast<int>(L->e_begin);
    pa.e_end = static_cast<int>(L->e_end);
    pa.num_shared = with_shared ? static_cast<int>(g.S) : 0;
    pa.mb_count = static_cast<int>(g.mb_count);
    pa.kc_total = cf.kc_total;
    pa.nsplit = nsplit;
    pa.nsplit_min = ns_min;
    {
        // one more K split writes (and the combine re-reads) another f32 partial of every
        // routed row; weigh it against the residual payload the GEMM must stream anyway
        const int64_t local = L->e_end - L->e_begin;
        const double active = static_cast<double>(std::min<int64_t>(local, batch * g.top_k) + g.S);
        const double wbytes = active * static_cast<double>(g.o) * static_cast<double>(g.i) * g.bits / 8.0;
        const double obytes = static_cast<double>(compact_rows(L, batch)) * static_cast<double>(g.o) * 8.0;
        pa.split_cost = static_cast<float>(obytes / std::max(1.0, wbytes));
    }
    pa.run_order = xr ? 1 : 0;
    {
        // ext-balanced K splits: opt-in (TQ_EXT_BALANCE=1) -- measured slower on the
        // c2 sweep (739 vs 717 us): the per-unit chain, not the ext bytes, bounds the
        // last split's CTAs, and uneven main-chunk counts cost more than they save
        constexpr bool ext_balance = false;
        if (ext_balance && use_qmoe && cf.n_ext > 0 && g.ext_cols > 0) {
            // ext blocks (dense fp16, 128 x 64 per block) against one packed main chunk
            const double ext_bytes = static_cast<double>(g.ext_cols) * kBM * 2.0;
            const double chunk_bytes = static_cast<double>(cf.kc) * kBM * g.bits / 8.0 + kBM * 2.0;
            pa.ext8 = static_cast<int>(8.0 * ext_bytes / chunk_bytes + 0.5);
        }
        pa.max_run = xr ? xr_slots(cf, ns_min) : 0;
        // per-unit pipeline cost of the decode GEMM in chunk equivalents (TQ_PROFILE:
        // ~1 us per unit vs ~0.27 us per 6.9 KB chunk)
        constexpr int unit_cost8 = 30;
        pa.unit_cost8 = (xr && use_qmoe) ? unit_cost8 : 0;
    }
    pa.n_ext = cf.n_ext;
    pa.main_kc = use_qmoe ? 1 : 0;
    pa.num_sms = L->num_sms;
    pa.bn = cf.bn;
    pa.proj_bn = cfp.bn;
    pa.nsplit_out = L->nsplit_d.as<int32_t>();
    pa.proj_mb = use_lotile ? static_cast<int>(L->proj_mb) : 0;
    pa.proj_kc_total = cfp.kc_total;
    pa.proj_nsplit = pns;
    pa.perm = L->perm.as<int32_t>();
    pa.inv = L->inv.as<int32_t>();
    pa.offsets = L->offsets.as<int32_t>();
    pa.poffsets = L->poffsets.as<int32_t>();
    pa.units = L->units.as<Unit>();
    pa.n_units = L->n_units.as<int32_t>();
    pa.proj_units = L->punits.as<Unit>();
    pa.n_proj_units = L->n_punits.as<int32_t>();
    pa.err_flag = L->err_flag.as<int32_t>();
    return pa;
}

// plan_done: the router already ran the plan (run_route with make_plan_args)
void run_experts(tq_layer* L, const float* x, int64_t batch, const int32_t* ids, const float* gates, float* y,
                 int path, cudaStream_t st) {
    (void)x;
    const Geometry& g = L->g;
    const bool use_lotile = path != TQ_PATH_QMOE;
    const bool use_qmoe = path != TQ_PATH_LOTILE;
    const LaunchCfg cf = main_cfg(L, batch, path);
    const LaunchCfg cfp = proj_cfg(L, batch);
    const bool xr = cf.dn == 32;
    const int ns_min = use_qmoe ? xr_ns_min(L, cf, batch) : 1;
    const int pns = proj_nsplit(L, batch);
    const bool with_shared = use_qmoe && g.S > 0;
    const PlanArgs pa = make_plan_args(L, batch, ids, path);
    cuda_check(launch_plan(pa, st), "plan_kernel launch");
    count_launch(L);
    const int64_t atom_rows = rows_for(L, L->cap);   // capacity rows of xperm / extperm / ypart
    // projection pass: Z = P . x for every token (dense fp16 weights)
    if (use_lotile && L->proj_mb > 0) {
        GemmParams p = base_params(L, cfp, batch);
        p.tmap_x64 = L->map_x16_64;
        p.tmap_e64 = L->map_x16_64;
        p.tmap_x16 = L->map_x16_16;
        p.tmap_e16 = L->map_x16_16;
        p.x_ptr = L->x16.as<__half>();
        p.x_ld = g.k_pad;
        p.e_ptr = L->x16.as<__half>();
        p.e_ld = g.k_pad;
        p.codes = L->pcodes.as<uint8_t>();
        p.weight_stride = L->pweight_stride;
        p.w_outscale = L->p_outscale.as<float>();
        p.units = L->punits.as<Unit>();
        p.n_units = L->n_punits.as<int32_t>();
        p.y = L->zpart.as<float>();
        p.y_split_stride = batch * L->proj_rows;
        p.ldy = static_cast<int32_t>(L->proj_rows);
        p.o_valid = static_cast<int32_t>(L->proj_rows);
        p.o_pad = static_cast<int32_t>(L->proj_o_pad);
        p.bits = kDenseBits;
        p.groups = 0;
        p.rank = 0;
        const int64_t nunits = L->proj_mb * ((batch + cfp.bn - 1) / cfp.bn) * pns;
        cuda_check(launch_gemm(p, static_cast<int>(std::min<int64_t>(nunits, L->num_sms)), st), "projection gemm launch");
        count_launch(L);
    }
    // gather
    GatherArgs ga{};
    ga.x16 = L->x16.as<__half>();
    ga.sx = L->sx.as<float>();
    ga.zpart = L->zpart.as<float>();
    ga.zsplit_stride = batch * L->proj_rows;
    ga.zcols = static_cast<int>(L->proj_rows);
    ga.proj_nsplit = pns;
    ga.ids = ids;
    ga.perm = L->perm.as<int32_t>();
    ga.offsets = L->offsets.as<int32_t>();
    ga.pm_of = L->pm_of.as<int32_t>();
    ga.zscale = L->zscale.as<float>();
    ga.rowscale = L->rowscale.as<float>();
    ga.batch = static_cast<int>(batch);
    ga.top_k = static_cast<int>(g.top_k);
    ga.num_experts = static_cast<int>(g.K);
    ga.k_pad = static_cast<int>(g.k_pad);
    ga.groups = static_cast<int>(g.G);
    ga.rank = static_cast<int>(g.r);
    ga.ext_cols = static_cast<int>(g.ext_cols);
    ga.with_shared = with_shared ? 1 : 0;
    ga.use_sx = use_qmoe ? 1 : 0;
    ga.use_z = (use_lotile && L->proj_mb > 0) ? 1 : 0;
    ga.xp = L->xperm.as<__half>();
    ga.ep = L->extperm.as<__half>();
    ga.poffsets = L->poffsets.as<int32_t>();
    ga.atom_rows = atom_rows;
    ga.inv = L->inv.as<int32_t>();
    cuda_check(launch_gather_tokens(ga, st), "gather_tokens_kernel launch");
    count_launch(L);
    // fused expert pass
    GemmParams p = base_params(L, cf, batch);
    p.tmap_x64 = L->map_xp64;
    p.tmap_e64 = L->map_ep64;
    p.tmap_x16 = L->map_xp16;
    p.tmap_e16 = L->map_ep16;
    p.x_ptr = L->xperm.as<__half>();
    p.x_ld = g.k_pad;
    p.e_ptr = L->extperm.as<__half>();
    p.e_ld = g.ext_cols;
    p.x_atom_rows = atom_rows;
    p.contig = xr ? 1 : 0;
    p.e_slots = xr ? 1 : 2;
    p.xr_slots = xr ? (use_qmoe ? xr_slots(cf, ns_min) : std::max(1, cf.n_ext)) : 0;   // lotile-only units: ext chunks only
    p.codes = L->codes.as<uint8_t>();
    p.weight_stride = L->weight_stride;
    p.scales = L->scales.as<__half>();
    p.ext_blocks = L->ext_blocks.as<uint8_t>();
    p.n_ext64 = static_cast<int32_t>(L->g.n_ext);
    p.w_outscale = L->w_outscale.as<float>();
    p.units = L->units.as<Unit>();
    p.n_units = L->n_units.as<int32_t>();
    p.y = L->ypart.as<float>();
    p.y_split_stride = rows_for(L, batch) * g.o;
    p.ldy = static_cast<int32_t>(g.o);
    p.o_valid = static_cast<int32_t>(g.o);
    p.o_pad = static_cast<int32_t>(g.o_pad);
    p.bits = g.bits;
    p.groups = static_cast<int32_t>(g.G);
    p.rank = static_cast<int32_t>(g.r);
    // (an epilogue-fused combine -- red.global.add of at most two addends per output --
    // was measured slower at prefill than this separate combine pass)
    timed_expert_gemm(L, p, L->num_sms, st);
    count_launch(L);
    // combine
    CombineArgs ca{};
    ca.y = L->ypart.as<float>();
    ca.split_stride = rows_for(L, batch) * g.o;
    ca.nsplit = pa.nsplit;
    ca.inv = L->inv.as<int32_t>();
    ca.gates = gates;
    ca.offsets = L->offsets.as<int32_t>();
    ca.ids = ids;
    ca.poffsets = L->poffsets.as<int32_t>();
    ca.num_experts = static_cast<int>(g.K);
    ca.batch = static_cast<int>(batch);
    ca.top_k = static_cast<int>(g.top_k);
    ca.out_dim = static_cast<int>(g.o);
    ca.num_shared = with_shared ? static_cast<int>(g.S) : 0;
    ca.use_routed = 1;
    ca.ysh = L->ypart.as<float>();
    ca.sh_split_stride = ca.split_stride;
    ca.sh_nsplit = pa.nsplit;
    ca.sh_from_offsets = 1;
    ca.nsplit_dev = L->nsplit_d.as<int32_t>();
    ca.out = y;
    cuda_check(launch_combine(ca, st), "combine_kernel launch");
    count_launch(L);
}

// ---------------------------------------------------------------------------
// decode path: 3 launches per forward (route+project+scatter, fused expert GEMM
// with split-segment fixup, combine)
// ---------------------------------------------------------------------------
constexpr int64_t kDecMaxBatch = 256;  // slots per expert (and tokens) the decode workspace holds

bool decode_ok(const tq_layer* L, int64_t batch, bool given) {
    const Geometry& g = L->g;
    const int64_t slots = given ? batch * g.top_k : batch;
    return !L->dense && batch > 0 && slots <= kDecMaxBatch && g.top_k <= kDecMaxTopK && g.K <= 64 &&
           g.K + g.S <= kDecMaxW && L->e_begin == 0 && L->e_end == g.K && g.r <= 64 && g.G <= 64 && g.n_ext <= 4;
}

void reserve_decode(tq_layer* L) {
    if (L->dec_ready) return;
    cuda_check(cudaSetDevice(L->device), "cudaSetDevice");
    const Geometry& g = L->g;
    const int64_t W = g.K + g.S;
    const int64_t rows = W * kDecMaxBatch + 64;   // + slack: 16-row MMA tiles read past a weight's last slot
    L->dec_atom_rows = rows;
    L->dec_xperm.alloc(sizeof(__half) * rows * g.k_pad);
    L->dec_extperm.alloc(sizeof(__half) * rows * g.n_ext * 64);
    cuda_check(cudaMemset(L->dec_xperm.p, 0, L->dec_xperm.n), "cudaMemset");
    cuda_check(cudaMemset(L->dec_extperm.p, 0, L->dec_extperm.n), "cudaMemset");
    L->dec_yslot.alloc(sizeof(float) * W * kDecMaxBatch * g.o);
    L->dec_cnt.alloc(sizeof(int32_t) * g.K);
    cuda_check(cudaMemset(L->dec_cnt.p, 0, L->dec_cnt.n), "cudaMemset");
    L->dec_inv.alloc(sizeof(int32_t) * kDecMaxBatch * g.top_k);
    L->dec_zq.alloc(sizeof(float) * kDecMaxBatch * g.N * g.r);
    L->dec_scratch.alloc(sizeof(float) * L->num_sms * 2 * 64 * kBM);
    L->dec_segcnt.alloc(sizeof(int32_t) * W * ((kDecMaxBatch + 63) / 64) * g.mb_count);
    cuda_check(cudaMemset(L->dec_segcnt.p, 0, L->dec_segcnt.n), "cudaMemset");
    L->dec_ticket.alloc(sizeof(int32_t) * kDecMaxBatch);   // the decode router's own per-token tickets
    cuda_check(cudaMemset(L->dec_ticket.p, 0, L->dec_ticket.n), "cudaMemset");
    L->dec_ready = true;
}

// ids_in / gates_in: given routing (tq_forward) or null (routed here)
void run_decode(tq_layer* L, const float* x, int64_t batch, const int32_t* ids_in, const float* gates_in, float* y,
                int path, cudaStream_t st) {
    const Geometry& g = L->g;
    reserve_decode(L);
    const bool given = ids_in != nullptr;
    const bool use_main = path != TQ_PATH_LOTILE;
    const bool use_lr = path != TQ_PATH_QMOE;
    const int S = use_main ? static_cast<int>(g.S) : 0;   // lotile_forward has no shared experts
    const int64_t cap8 = round_up(given ? batch * g.top_k : batch, 8);
    // 32-slot tiles (4 MMA issue streams) up to 64 slots per weight: at uniform routing an
    // expert of a 64-token batch holds ~16 slots, and the 2-issuer 64-slot tile pays
    // twice the per-MMA issue latency per step; an expert past 32 slots takes two tiles
    const int dn = cap8 <= 64 ? 32 : 64;
    if (L->ktime) {
        L->kt_stream = st;
        L->kt_active = true;
        cudaEvent_t e;
        cudaEventCreate(&e);
        cudaEventRecord(e, st);
        L->kev.push_back({e});
    }
    DecRouteArgs ra{};
    ra.x = x;
    ra.batch = static_cast<int>(batch);
    ra.in_dim = static_cast<int>(g.i);
    ra.k_pad = static_cast<int>(g.k_pad);
    ra.gate = L->gate.as<float>();
    ra.num_experts = static_cast<int>(g.K);
    ra.top_k = static_cast<int>(g.top_k);
    ra.num_shared = S;
    ra.given = given ? 1 : 0;
    ra.ids_in = ids_in;
    ra.ids = L->ids.as<int32_t>();
    ra.gates = L->gates.as<float>();
    ra.score_ws = L->route_ws.as<float>();
    ra.ticket = L->dec_ticket.as<int32_t>();
    ra.group_size = static_cast<int>(g.gs);
    ra.groups = static_cast<int>(g.G);
    ra.rank = static_cast<int>(g.r);
    ra.num_q = static_cast<int>(g.N);
    ra.vcodes = L->vcodes.as<int8_t>();
    ra.vscale = L->vscale.as<float>();
    ra.q_tier = L->q_tier.as<int32_t>();
    ra.q_first = L->q_first.as<int32_t>();
    ra.scaling = L->scaling_d.as<float>();
    ra.e_q = L->e_q.as<int32_t>();
    ra.zscale = L->zscale.as<float>();
    ra.zq_ws = L->dec_zq.as<float>();
    ra.use_main = use_main ? 1 : 0;
    ra.use_lr = use_lr ? 1 : 0;
    ra.cap8 = static_cast<int>(cap8);
    ra.atom_rows = L->dec_atom_rows;
    ra.ext_cols = static_cast<int>(g.n_ext * 64);
    ra.xperm = L->dec_xperm.as<__half>();
    ra.extperm = L->dec_extperm.as<__half>();
    ra.cnt = L->dec_cnt.as<int32_t>();
    ra.inv = L->dec_inv.as<int32_t>();
    ra.err_flag = L->err_flag.as<int32_t>();
#ifdef TQ_ROUTE_TRACE
    static unsigned long long* rbuf = nullptr;
    const size_t rbytes = sizeof(unsigned long long) * 16 * 64 * 128;
    if (!rbuf) cuda_check(cudaMalloc(&rbuf, rbytes), "cudaMalloc");
    cuda_check(cudaMemsetAsync(rbuf, 0, rbytes, st), "cudaMemset");
    ra.trace = rbuf;
#endif
    cuda_check(launch_dec_route(ra, st), "dec_route_kernel launch");
#ifdef TQ_ROUTE_TRACE
    if (getenv("TQ_ROUTE_TRACE_FILE")) {
        std::vector<unsigned long long> hb(16 * 64 * 128);
        cuda_check(cudaStreamSynchronize(st), "sync");
        cuda_check(cudaMemcpy(hb.data(), rbuf, rbytes, cudaMemcpyDeviceToHost), "trace D2H");
        if (FILE* f = fopen(getenv("TQ_ROUTE_TRACE_FILE"), "ab")) {
            fwrite(hb.data(), 8, hb.size(), f);
            fclose(f);
        }
    }
#endif
    count_launch(L);

    DecParams dp{};
    dp.codes = L->codes.as<uint8_t>();
    dp.weight_stride = L->weight_stride;
    dp.scales = L->scales.as<__half>();
    dp.ext_blocks = L->ext_blocks.as<uint8_t>();
    dp.n_ext64 = static_cast<int>(g.n_ext);
    dp.w_outscale = L->w_outscale.as<float>();
    dp.bits = static_cast<int>(g.bits);
    dp.group_size = static_cast<int>(g.gs);
    dp.groups = static_cast<int>(g.G);
    dp.kc64 = static_cast<int>(g.kc_total);
    dp.nmain = use_main ? static_cast<int>((g.kc_total + 3) / 4) : 0;   // 256-K steps
    dp.mb_count = static_cast<int>(g.mb_count);
    dp.o_valid = static_cast<int>(g.o);
    dp.num_experts = static_cast<int>(g.K);
    dp.num_shared = S;
    dp.batch = static_cast<int>(batch);
    dp.cnt = L->dec_cnt.as<int32_t>();
    dp.cap8 = static_cast<int>(cap8);
    dp.atom_rows = L->dec_atom_rows;
    dp.xperm = L->dec_xperm.as<__half>();
    dp.extperm = L->dec_extperm.as<__half>();
    dp.yslot = L->dec_yslot.as<float>();
    dp.ldy = static_cast<int>(g.o);
    dp.scratch = L->dec_scratch.as<float>();
    dp.seg_cnt = L->dec_segcnt.as<int32_t>();
    dp.check_slots = static_cast<int>(batch * g.top_k);
    {
        cudaEvent_t ev0 = nullptr, ev1 = nullptr;
        if (L->timing) {
            cuda_check(cudaEventCreate(&ev0), "cudaEventCreate");
            cuda_check(cudaEventCreate(&ev1), "cudaEventCreate");
            cuda_check(cudaEventRecord(ev0, st), "cudaEventRecord");
        }
#ifdef TQ_DEC_TRACE
        // diagnostics build: event trace of one CTA, dumped to $TQ_DEC_TRACE_FILE after each launch
        static unsigned long long* tbuf = nullptr;
        if (!tbuf) cuda_check(cudaMalloc(&tbuf, 16 * 1024 * 8), "cudaMalloc");
        cuda_check(cudaMemsetAsync(tbuf, 0, 16 * 1024 * 8, st), "cudaMemset");   // [10][1024] events | [148][4] per CTA at 12288
        dp.trace = tbuf;
        dp.trace_cta = getenv("TQ_DEC_TRACE_CTA") ? atoi(getenv("TQ_DEC_TRACE_CTA")) : 0;
#endif
        cuda_check(launch_decode(dp, dn, L->num_sms, st), "dec_gemm_kernel launch");
#ifdef TQ_DEC_TRACE
        if (getenv("TQ_DEC_TRACE_FILE")) {
            std::vector<unsigned long long> hbuf(16 * 1024);
            cuda_check(cudaStreamSynchronize(st), "sync");
            cuda_check(cudaMemcpy(hbuf.data(), tbuf, 16 * 1024 * 8, cudaMemcpyDeviceToHost), "trace D2H");
            if (FILE* f = fopen(getenv("TQ_DEC_TRACE_FILE"), "ab")) {
                fwrite(hbuf.data(), 8, hbuf.size(), f);
                fclose(f);
            }
        }
#endif
        if (L->timing) {
            cuda_check(cudaEventRecord(ev1, st), "cudaEventRecord");
            L->tev.emplace_back(ev0, ev1);
        }
    }
    count_launch(L);

    DecCombineArgs ca{};
    ca.yslot = L->dec_yslot.as<float>();
    ca.ldy = static_cast<int>(g.o);
    ca.inv = L->dec_inv.as<int32_t>();
    ca.gates = given ? gates_in : L->gates.as<float>();
    ca.batch = static_cast<int>(batch);
    ca.top_k = static_cast<int>(g.top_k);
    ca.out_dim = static_cast<int>(g.o);
    ca.num_shared = S;
    ca.num_experts = static_cast<int>(g.K);
    ca.cap8 = static_cast<int>(cap8);
    ca.cnt = L->dec_cnt.as<int32_t>();
    ca.out = y;
    cuda_check(launch_dec_combine(ca, st), "dec_combine_kernel launch");
    count_launch(L);
}

void check_layer(const tq_layer* L) {
    if (!L) fail(TQ_ERR_PARAM, "null layer");
}

void check_batch(tq_layer* L, int64_t batch) {
    if (batch < 0) fail(TQ_ERR_SHAPE, "negative batch");
    if (batch > L->cap) reserve(L, batch);
    if (L->e_begin != 0 || L->e_end != L->g.K)
        fail(TQ_ERR_PARAM, "layer holds only experts [" + std::to_string(L->e_begin) + ", " + std::to_string(L->e_end) +
                               "); use the expert-parallel entry points");
}

}  // namespace

// ---------------------------------------------------------------------------
// C-ABI
// ---------------------------------------------------------------------------

namespace {
// Run `body` (which enqueues a forward on the stream it is given) through the
// layer's graph cache: captured once per argument set on a private stream,
// then replayed on the caller's stream with one cudaGraphLaunch.
template <class Body>
void run_graphed(tq_layer* L, const void* const (&key)[6], int64_t batch, int path, cudaStream_t st, Body body) {
    if (!L->use_graphs || L->timing || L->ktime) {
        body(st);
        return;
    }
    tq_layer::GraphEntry* hit = nullptr;
    for (auto& g : L->graphs)
        if (g.batch == batch && g.path == path && std::equal(key, key + 6, g.key)) hit = &g;
    if (!hit) {
        if (!L->cap_stream)
            cuda_check(cudaStreamCreateWithFlags(&L->cap_stream, cudaStreamNonBlocking), "cudaStreamCreate");
        if (L->graphs.size() >= 64) L->drop_graphs();
        const uint64_t before = L->launches;
        cudaGraph_t graph = nullptr;
        cuda_check(cudaStreamBeginCapture(L->cap_stream, cudaStreamCaptureModeThreadLocal), "cudaStreamBeginCapture");
        try {
            body(L->cap_stream);
        } catch (...) {
            cudaStreamEndCapture(L->cap_stream, &graph);
            if (graph) cudaGraphDestroy(graph);
            throw;
        }
        cuda_check(cudaStreamEndCapture(L->cap_stream, &graph), "cudaStreamEndCapture");
        tq_layer::GraphEntry e{};
        std::copy(key, key + 6, e.key);
        e.batch = batch;
        e.path = path;
        e.launches = L->launches - before;
        L->launches = before;
        const cudaError_t ie = cudaGraphInstantiate(&e.exec, graph, 0);
        cudaGraphDestroy(graph);
        cuda_check(ie, "cudaGraphInstantiate");
        L->graphs.push_back(e);
        hit = &L->graphs.back();
    }
    cuda_check(cudaGraphLaunch(hit->exec, st), "cudaGraphLaunch");
    L->launches += hit->launches;
}
}  // namespace

extern "C" {

const char* tq_last_error(void) { return g_last_error.c_str(); }

const char* tq_version(void) { return "tileq_b200 0.1 (sm_100a, tcgen05 TS grouped GEMM)"; }

tq_status tq_layer_load(const char* dir, int device, int verify_crc, int64_t expert_begin, int64_t expert_end,
                        tq_layer** out) {
    return guarded([&] {
        if (!dir || !out) fail(TQ_ERR_PARAM, "tq_layer_load: null argument");
        HostArtifact a = read_artifact_dir(dir, verify_crc != 0);
        auto L = std::make_unique<tq_layer>();
        build_layer(L.get(), a, device, expert_begin, expert_end);
        *out = L.release();
    });
}

tq_status tq_artifact_check(const char* dir, int verify_crc) {
    return guarded([&] {
        if (!dir) fail(TQ_ERR_PARAM, "tq_artifact_check: null argument");
        HostArtifact a = read_artifact_dir(dir, verify_crc != 0);
        check_host_artifact(a);
    });
}

tq_status tq_layer_create(const tq_layer_desc* desc, int device, int64_t expert_begin, int64_t expert_end,
                          tq_layer** out) {
    return guarded([&] {
        if (!desc || !out) fail(TQ_ERR_PARAM, "tq_layer_create: null argument");
        HostArtifact a = artifact_from_desc(desc);
        auto L = std::make_unique<tq_layer>();
        build_layer(L.get(), a, device, expert_begin, expert_end);
        *out = L.release();
    });
}

tq_status tq_layer_free(tq_layer* layer) {
    return guarded([&] {
        if (layer) {
            cudaSetDevice(layer->device);
            delete layer;
        }
    });
}

tq_status tq_layer_info_get(const tq_layer* L, tq_layer_info* out) {
    return guarded([&] {
        check_layer(L);
        out->num_experts = L->g.K;
        out->top_k = L->g.top_k;
        out->in_dim = L->g.i;
        out->out_dim = L->g.o;
        out->num_shared = L->g.S;
        out->rank = L->g.r;
        out->grid_rows = L->g.M;
        out->grid_cols = L->g.N;
        out->bits = L->dense ? L->art_bits : L->g.bits;
        out->group_size = L->dense ? L->art_gs : L->g.gs;
        out->expert_begin = L->e_begin;
        out->expert_end = L->e_end;
        out->device = L->device;
        out->device_bytes = L->device_bytes;
        out->tier_folded = L->tiers[0];
        out->tier_scalar = L->tiers[1];
        out->tier_general = L->tiers[2];
    });
}

tq_status tq_layer_reserve(tq_layer* L, int64_t max_tokens) {
    return guarded([&] {
        check_layer(L);
        reserve(L, max_tokens);
    });
}

tq_status tq_route(tq_layer* L, const float* x, int64_t batch, int32_t* ids, float* gates, void* stream) {
    return guarded([&] {
        check_layer(L);
        if (batch < 0) fail(TQ_ERR_SHAPE, "negative batch");
        if (batch == 0) return;
        if (batch > L->cap) reserve(L, batch);
        cuda_check(cudaSetDevice(L->device), "cudaSetDevice");
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        run_route(L, x, batch, true, st);
        cuda_check(cudaMemcpyAsync(ids, L->ids.p, sizeof(int32_t) * batch * L->g.top_k, cudaMemcpyDeviceToDevice, st),
                   "ids copy");
        cuda_check(cudaMemcpyAsync(gates, L->gates.p, sizeof(float) * batch * L->g.top_k, cudaMemcpyDeviceToDevice, st),
                   "gates copy");
    });
}

tq_status tq_permute(tq_layer* L, const int32_t* ids, int64_t batch, int32_t* perm, int32_t* offsets, int32_t* inv,
                     void* stream) {
    return guarded([&] {
        check_layer(L);
        if (batch < 0) fail(TQ_ERR_SHAPE, "negative batch");
        if (batch > L->cap) reserve(L, batch);
        cuda_check(cudaSetDevice(L->device), "cudaSetDevice");
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        PlanArgs pa{};
        pa.ids = ids;
        pa.batch = static_cast<int>(batch);
        pa.top_k = static_cast<int>(L->g.top_k);
        pa.num_experts = static_cast<int>(L->g.K);
        pa.e_begin = 0;
        pa.e_end = 0;
        pa.mb_count = static_cast<int>(L->g.mb_count);
        pa.kc_total = static_cast<int>(L->g.kc_total);
        pa.nsplit = 1;
        pa.num_sms = L->num_sms;
        pa.bn = gemm_dn_host(64);
        pa.perm = perm;
        pa.inv = inv;
        pa.offsets = offsets;
        pa.units = L->units.as<Unit>();
        pa.n_units = L->n_units.as<int32_t>();
        pa.proj_units = L->punits.as<Unit>();
        pa.n_proj_units = nullptr;
        pa.err_flag = L->err_flag.as<int32_t>();
        cuda_check(launch_plan(pa, st), "plan_kernel launch");
        count_launch(L);
    });
}


tq_status tq_forward(tq_layer* L, const float* x, int64_t batch, const int32_t* ids, const float* gates, float* y,
                     int path, void* stream) {
    return guarded([&] {
        check_layer(L);
        if (path < 0 || path > 2) fail(TQ_ERR_PARAM, "unknown path " + std::to_string(path));
        check_batch(L, batch);
        if (batch == 0) return;
        cuda_check(cudaSetDevice(L->device), "cudaSetDevice");
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        const void* const key[6] = {x, ids, gates, y, nullptr, nullptr};
        const bool dec = decode_ok(L, batch, true);
        if (dec) reserve_decode(L);
        run_graphed(L, key, batch, path + (dec ? 64 : 0), st, [&](cudaStream_t s2) {
            if (dec) {
                run_decode(L, x, batch, ids, gates, y, path, s2);
                return;
            }
            run_route(L, x, batch, false, s2);
            run_experts(L, x, batch, ids, gates, y, path, s2);
        });
    });
}

tq_status tq_forward_routed(tq_layer* L, const float* x, int64_t batch, float* y, int32_t* ids, float* gates, int path,
                            void* stream) {
    return guarded([&] {
        check_layer(L);
        if (path < 0 || path > 2) fail(TQ_ERR_PARAM, "unknown path " + std::to_string(path));
        check_batch(L, batch);
        if (batch == 0) return;
        cuda_check(cudaSetDevice(L->device), "cudaSetDevice");
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        const void* const key[6] = {x, nullptr, nullptr, y, ids, gates};
        const bool dec = decode_ok(L, batch, false);
        if (dec) reserve_decode(L);
        run_graphed(L, key, batch, path + 16, st, [&](cudaStream_t s2) {
            if (dec) {
                run_decode(L, x, batch, nullptr, nullptr, y, path, s2);
            } else {
                run_route(L, x, batch, true, s2);
                run_experts(L, x, batch, L->ids.as<int32_t>(), L->gates.as<float>(), y, path, s2);
            }
            if (ids)
                cuda_check(cudaMemcpyAsync(ids, L->ids.p, sizeof(int32_t) * batch * L->g.top_k, cudaMemcpyDeviceToDevice,
                                           s2),
                           "ids copy");
            if (gates)
                cuda_check(cudaMemcpyAsync(gates, L->gates.p, sizeof(float) * batch * L->g.top_k,
                                           cudaMemcpyDeviceToDevice, s2),
                           "gates copy");
        });
    });
}

tq_status tq_forward_host(tq_layer* L, const float* x, int64_t batch, float* y, int64_t* ids, float* gates, int path) {
    return guarded([&] {
        check_layer(L);
        if (path < 0 || path > 2) fail(TQ_ERR_PARAM, "unknown path " + std::to_string(path));
        check_batch(L, batch);
        if (batch == 0) return;
        cuda_check(cudaSetDevice(L->device), "cudaSetDevice");
        cudaStream_t st = nullptr;
        const bool dec = decode_ok(L, batch, false);
        if (dec) reserve_decode(L);
        auto body = [&](cudaStream_t s2) {
            cuda_check(cudaMemcpyAsync(L->xin.p, x, sizeof(float) * batch * L->g.i, cudaMemcpyHostToDevice, s2), "x H2D");
            if (dec) {
                run_decode(L, L->xin.as<float>(), batch, nullptr, nullptr, L->yout.as<float>(), path, s2);
            } else {
                run_route(L, L->xin.as<float>(), batch, true, s2);
                run_experts(L, L->xin.as<float>(), batch, L->ids.as<int32_t>(), L->gates.as<float>(),
                            L->yout.as<float>(), path, s2);
            }
            cuda_check(cudaMemcpyAsync(y, L->yout.p, sizeof(float) * batch * L->g.o, cudaMemcpyDeviceToHost, s2),
                       "y D2H");
        };
        // page-locked host buffers: the copies and kernels replay as one CUDA graph
        auto pinned = [](const void* ptr) {
            cudaPointerAttributes at{};
            if (cudaPointerGetAttributes(&at, ptr) != cudaSuccess) {
                cudaGetLastError();
                return false;
            }
            return at.type == cudaMemoryTypeHost;
        };
        if (pinned(x) && pinned(y)) {
            const void* const key[6] = {x, y, nullptr, nullptr, nullptr, nullptr};
            run_graphed(L, key, batch, path + 32 + (dec ? 64 : 0), st, body);
        } else {
            body(st);
        }
        std::vector<int32_t> hid;
        if (ids) {
            hid.resize(static_cast<size_t>(batch * L->g.top_k));
            cuda_check(cudaMemcpyAsync(hid.data(), L->ids.p, sizeof(int32_t) * hid.size(), cudaMemcpyDeviceToHost, st),
                       "ids D2H");
        }
        if (gates)
            cuda_check(cudaMemcpyAsync(gates, L->gates.p, sizeof(float) * batch * L->g.top_k, cudaMemcpyDeviceToHost, st),
                       "gates D2H");
        cuda_check(cudaStreamSynchronize(st), "stream sync");
        for (size_t t = 0; t < hid.size(); ++t) ids[t] = hid[t];
    });
}

tq_status tq_forward_host_ids(tq_layer* L, const float* x, int64_t batch, const int64_t* ids, const float* gates,
                              float* y, int path) {
    return guarded([&] {
        check_layer(L);
        if (path < 0 || path > 2) fail(TQ_ERR_PARAM, "unknown path " + std::to_string(path));
        check_batch(L, batch);
        if (batch == 0) return;
        if (!x || !ids || !gates || !y) fail(TQ_ERR_PARAM, "tq_forward_host_ids: null argument");
        const int64_t n = batch * L->g.top_k;
        std::vector<int32_t> hid(static_cast<size_t>(n));
        for (int64_t t = 0; t < n; ++t) {
            if (ids[t] < 0 || ids[t] >= L->g.K)
                fail(TQ_ERR_PARAM, "reference_forward: expert id " + std::to_string(ids[t]) + " out of range [0, " +
                                       std::to_string(L->g.K) + ")");
            hid[static_cast<size_t>(t)] = static_cast<int32_t>(ids[t]);
        }
        cuda_check(cudaSetDevice(L->device), "cudaSetDevice");
        if (L->hids.n < sizeof(int32_t) * static_cast<size_t>(n)) {
            L->hids.alloc(sizeof(int32_t) * static_cast<size_t>(L->cap * L->g.top_k));
            L->hgates.alloc(sizeof(float) * static_cast<size_t>(L->cap * L->g.top_k));
        }
        cudaStream_t st = nullptr;
        cuda_check(cudaMemcpyAsync(L->xin.p, x, sizeof(float) * batch * L->g.i, cudaMemcpyHostToDevice, st), "x H2D");
        cuda_check(cudaMemcpyAsync(L->hids.p, hid.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice, st), "ids H2D");
        cuda_check(cudaMemcpyAsync(L->hgates.p, gates, sizeof(float) * n, cudaMemcpyHostToDevice, st), "gates H2D");
        const float* xd = L->xin.as<float>();
        const int32_t* idd = L->hids.as<int32_t>();
        const float* gd = L->hgates.as<float>();
        float* yd = L->yout.as<float>();
        const void* const key[6] = {xd, idd, gd, yd, nullptr, nullptr};
        const bool dec = decode_ok(L, batch, true);
        if (dec) reserve_decode(L);
        run_graphed(L, key, batch, path + (dec ? 64 : 0), st, [&](cudaStream_t s2) {
            if (dec) {
                run_decode(L, xd, batch, idd, gd, yd, path, s2);
                return;
            }
            run_route(L, xd, batch, false, s2);
            run_experts(L, xd, batch, idd, gd, yd, path, s2);
        });
        cuda_check(cudaMemcpyAsync(y, L->yout.p, sizeof(float) * batch * L->g.o, cudaMemcpyDeviceToHost, st), "y D2H");
        cuda_check(cudaStreamSynchronize(st), "stream sync");
    });
}

// ---------------------------------------------------------------------------
// comparison layouts (the paper's bench: infer.cpp:187-339, 345-426)
// ---------------------------------------------------------------------------

static void layout_prepare(tq_layer* L, int layout) {
    if (layout < 0 || layout > 3) fail(TQ_ERR_PARAM, "unknown layout " + std::to_string(layout));
    if (L->lay_ready[layout]) return;
    const Geometry& g = L->g;
    const int64_t O = g.o, I = g.i, R = L->lay.R;
    if ((layout == 1 || layout == 2) && !L->lay_U.p) L->lay_U.upload(L->lay.U.data(), sizeof(float) * L->lay.U.size());
    if (layout == 1) {
        // shared_1d_from_tiled_representative (infer.cpp:320-335): P = sigma * V_0, U_p(k) per expert
        std::vector<float> P(static_cast<size_t>(R * I));
        for (int64_t j = 0; j < R; ++j)
            for (int64_t c = 0; c < I; ++c)
                P[j * I + c] = static_cast<float>(static_cast<double>(L->lay.sigma[j]) * L->lay.V[j * I + c]);
        L->lay_proj1d.upload(P.data(), sizeof(float) * P.size());
    } else if (layout == 2) {
        // elementwise_factors_from_tiled (infer.cpp:271-289): right_k = V_q(k) / s_k, sigma at the product
        const int64_t nloc = L->e_end - L->e_begin;
        std::vector<float> right(static_cast<size_t>(nloc * R * I));
        for (int64_t k = 0; k < nloc; ++k) {
            const int64_t e = L->e_begin + k;
            const int64_t q = L->lay.placement[2 * e + 1];
            const float* v = L->lay.V.data() + q * R * I;
            const float* sk = L->lay.scaling.data() + e * I;
            for (int64_t j = 0; j < R; ++j)
                for (int64_t c = 0; c < I; ++c)
                    right[(k * R + j) * I + c] = static_cast<float>(static_cast<double>(v[j * I + c]) / sk[c]);
        }
        L->lay_right.upload(right.data(), sizeof(float) * right.size());
        L->lay_sigma.upload(L->lay.sigma.data(), sizeof(float) * L->lay.sigma.size());
    } else if (layout == 3) {
        L->lay_dq.alloc(sizeof(uint16_t) * static_cast<size_t>((L->e_end - L->e_begin) * O * I));
    }
    (void)O;
    L->lay_ready[layout] = true;
}

static void launch_dequant_experts(tq_layer* L, uint16_t* out, cudaStream_t st) {
    const Geometry& g = L->g;
    DequantAllArgs a{};
    a.codes = L->codes.as<uint8_t>();
    a.weight_stride = L->weight_stride;
    a.scales = L->scales.as<uint16_t>();
    a.ext_blocks = L->ext_blocks.as<uint8_t>();
    a.ext_bytes = g.n_ext * code_block_bytes(kDenseBits);
    a.w_outscale = L->w_outscale.as<float>();
    a.out = reinterpret_cast<__half*>(out);
    a.o = g.o;
    a.i = g.i;
    a.n_weights = static_cast<int>(L->e_end - L->e_begin);
    a.mb_count = static_cast<int>(g.mb_count);
    a.kb_total = static_cast<int>(g.k_pad / kKC);
    a.groups = static_cast<int>(g.G);
    a.group_size = static_cast<int>(g.gs);
    cuda_check(launch_dequant_all(a, g.bits, st), "dequant_all_kernel launch");
    count_launch(L);
}

tq_status tq_layout_prepare(tq_layer* L, int layout) {
    return guarded([&] {
        check_layer(L);
        cuda_check(cudaSetDevice(L->device), "cudaSetDevice");
        layout_prepare(L, layout);
    });
}

tq_status tq_layout_forward(tq_layer* L, int layout, const float* x, int64_t batch, const int32_t* ids,
                            const float* gates, float* y, int64_t* dispatches, void* stream) {
    return guarded([&] {
        check_layer(L);
        check_batch(L, batch);
        cuda_check(cudaSetDevice(L->device), "cudaSetDevice");
        layout_prepare(L, layout);
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        const Geometry& g = L->g;
        const int64_t k = g.top_k, O = g.o, I = g.i, R = L->lay.R;
        int64_t disp = 0;
        if (layout == TQ_LAYOUT_FUSED_2D) {
            if (batch > 0) {
                run_route(L, x, batch, false, st);
                run_experts(L, x, batch, ids, gates, y, TQ_PATH_LOTILE, st);
            }
            disp = 2;   // the two fused products (infer.cpp:120,173)
        } else if (layout == TQ_LAYOUT_DEQUANT_ONLY) {
            launch_dequant_experts(L, L->lay_dq.as<uint16_t>(), st);
        } else {
            // host-orchestrated per-(token, expert) dispatches, as the reference loops
            std::vector<int32_t> h_ids(static_cast<size_t>(batch * k));
            if (batch > 0) {
                cuda_check(cudaMemcpyAsync(h_ids.data(), ids, sizeof(int32_t) * h_ids.size(), cudaMemcpyDeviceToHost, st),
                           "ids D2H");
                cuda_check(cudaStreamSynchronize(st), "cudaStreamSynchronize");
                cuda_check(cudaMemsetAsync(y, 0, sizeof(float) * batch * O, st), "y memset");
            }
            for (int32_t e : h_ids)
                if (e < L->e_begin || e >= L->e_end)
                    fail(TQ_ERR_PARAM, std::string(layout == 1 ? "1d" : "elementwise") + " baseline: expert id " +
                                           std::to_string(e) + " out of range");
            float* mid = L->zpart.as<float>();   // B*top_k x r scratch (>= cap * proj_rows floats)
            if (static_cast<int64_t>(L->zpart_cap_floats) < batch * k * R)
                fail(TQ_ERR_SIZE, "layout scratch too small: reserve a larger batch");
            if (layout == TQ_LAYOUT_SHARED_1D) {
                cuda_check(launch_lr_right(L->lay_proj1d.as<float>(), I, static_cast<int>(R), x, I,
                                           static_cast<int>(batch), static_cast<int>(I), nullptr, mid, R, st),
                           "shared projection launch");
                count_launch(L);
                disp = 1;
                for (int64_t b = 0; b < batch; ++b)
                    for (int64_t t = 0; t < k; ++t) {
                        const int64_t f = b * k + t;
                        const int64_t p = L->lay.placement[2 * h_ids[f]];
                        cuda_check(launch_lr_left(L->lay_U.as<float>() + p * O * R, static_cast<int>(O),
                                                  static_cast<int>(R), mid + b * R, gates + f, y + b * O, st),
                                   "output multiply launch");
                        count_launch(L);
                        ++disp;
                    }
            } else {
                for (int64_t b = 0; b < batch; ++b)
                    for (int64_t t = 0; t < k; ++t) {
                        const int64_t f = b * k + t;
                        const int64_t e = h_ids[f];
                        const int64_t p = L->lay.placement[2 * e];
                        cuda_check(launch_lr_right(L->lay_right.as<float>() + (e - L->e_begin) * R * I, I,
                                                   static_cast<int>(R), x + b * I, I, 1, static_cast<int>(I),
                                                   L->lay_sigma.as<float>(), mid + f * R, R, st),
                                   "right-factor multiply launch");
                        cuda_check(launch_lr_left(L->lay_U.as<float>() + p * O * R, static_cast<int>(O),
                                                  static_cast<int>(R), mid + f * R, gates + f, y + b * O, st),
                                   "left-factor multiply launch");
                        count_launch(L, 2);
                        disp += 2;
                    }
            }
        }
        if (dispatches) *dispatches = disp;
    });
}

tq_status tq_dequantize_experts(tq_layer* L, uint16_t* out, void* stream) {
    return guarded([&] {
        check_layer(L);
        cuda_check(cudaSetDevice(L->device), "cudaSetDevice");
        launch_dequant_experts(L, out, static_cast<cudaStream_t>(stream));
    });
}

// Diagnostics: the decode path's self-resetting device counters (slot counts, per
// token router tickets, split-segment arrivals), copied to the host; all must read
// zero between forwards.  out: [K] cnt, [cap] tickets, [(K + S) * mb_count] segments.
tq_status tq_debug_decode_counters(tq_layer* L, int32_t* out, int64_t n) {
    return guarded([&] {
        check_layer(L);
        cuda_check(cudaDeviceSynchronize(), "sync");
        const Geometry& g = L->g;
        std::vector<int32_t> h;
        auto pull = [&](const DBuf& b, int64_t cnt) {
            std::vector<int32_t> t(static_cast<size_t>(cnt), 0);
            if (b.p) cuda_check(cudaMemcpy(t.data(), b.p, sizeof(int32_t) * cnt, cudaMemcpyDeviceToHost), "D2H");
            h.insert(h.end(), t.begin(), t.end());
        };
        pull(L->dec_cnt, g.K);
        pull(L->dec_ticket, kDecMaxBatch);
        pull(L->dec_segcnt, (g.K + g.S) * g.mb_count);   // first tile of every weight
        for (int64_t t = 0; t < n && t < static_cast<int64_t>(h.size()); ++t) out[t] = h[static_cast<size_t>(t)];
    });
}

tq_status tq_exp_f64(const double* x, int64_t n, double* y, void* stream) {
    return guarded([&] {
        if (n < 0 || (n > 0 && (!x || !y))) fail(TQ_ERR_PARAM, "tq_exp_f64: bad arguments");
        cuda_check(launch_exp_f64(x, n, y, static_cast<cudaStream_t>(stream)), "exp launch");
    });
}

tq_status tq_sync(tq_layer* L, void* stream) {
    return guarded([&] {
        check_layer(L);
        cuda_check(cudaSetDevice(L->device), "cudaSetDevice");
        cuda_check(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)), "stream sync");
        int32_t flag = 0;
        cuda_check(cudaMemcpy(&flag, L->err_flag.p, sizeof(int32_t), cudaMemcpyDeviceToHost), "err flag D2H");
        if (flag) {
            cuda_check(cudaMemset(L->err_flag.p, 0, sizeof(int32_t)), "err flag reset");
            fail(TQ_ERR_PARAM, "reference_forward: expert id out of range [0, " + std::to_string(L->g.K) + ")");
        }
    });
}

tq_status tq_unpack_codes(const uint8_t* bytes, int64_t nbytes, int bits, int64_t count, uint32_t* out, void* stream) {
    return guarded([&] {
        if (bits != 2 && bits != 3 && bits != 4 && bits != 8)
            fail(TQ_ERR_PARAM, "bit packing supports widths {2,3,4,8}, got " + std::to_string(bits));
        if (count < 0 || static_cast<size_t>(nbytes) != packed_byte_length(static_cast<size_t>(count), bits))
            fail(TQ_ERR_PARAM, "packed stream holds " + std::to_string(nbytes) + " bytes, expected " +
                                   std::to_string(packed_byte_length(static_cast<size_t>(std::max<int64_t>(count, 0)), bits)) +
                                   " for " + std::to_string(count) + " codes at " + std::to_string(bits) + " bits");
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        int32_t* flag = nullptr;
        cuda_check(cudaMalloc(&flag, sizeof(int32_t)), "cudaMalloc");
        std::unique_ptr<int32_t, void (*)(int32_t*)> guard(flag, [](int32_t* f) { cudaFree(f); });
        cuda_check(cudaMemsetAsync(flag, 0, sizeof(int32_t), st), "memset");
        cuda_check(launch_unpack(bytes, nbytes, bits, count, out, flag, st), "unpack_kernel launch");
        int32_t h = 0;
        cuda_check(cudaMemcpyAsync(&h, flag, sizeof(int32_t), cudaMemcpyDeviceToHost, st), "flag D2H");
        cuda_check(cudaStreamSynchronize(st), "stream sync");
        if (h) fail(TQ_ERR_FORMAT, "packed stream has nonzero padding past code " + std::to_string(count));
    });
}

tq_status tq_layer_export_codes(tq_layer* L, int64_t e, uint32_t* out, void* stream) {
    return guarded([&] {
        check_layer(L);
        if (e < 0 || e >= L->n_weights) fail(TQ_ERR_PARAM, "export: matrix index out of range");
        if (L->dense) fail(TQ_ERR_PARAM, "export: this layer's residuals are resolved to fp16 weights at load; no codes kept");
        cuda_check(cudaSetDevice(L->device), "cudaSetDevice");
        cuda_check(launch_export_codes(L->codes.as<uint8_t>() + e * L->weight_stride, L->g.bits,
                                       static_cast<int>(L->g.kc_total), static_cast<int>(L->g.o),
                                       static_cast<int>(L->g.i), out, static_cast<cudaStream_t>(stream)),
                   "export launch");
    });
}

tq_status tq_gemm_timing_enable(tq_layer* L, int enable) {
    return guarded([&] {
        check_layer(L);
        cuda_check(cudaSetDevice(L->device), "cudaSetDevice");
        for (auto& e : L->tev) {
            cudaEventDestroy(e.first);
            cudaEventDestroy(e.second);
        }
        L->tev.clear();
        L->timing = enable != 0;
    });
}

tq_status tq_gemm_time_get(tq_layer* L, double* ms_total, int64_t* launches) {
    return guarded([&] {
        check_layer(L);
        cuda_check(cudaSetDevice(L->device), "cudaSetDevice");
        double tot = 0.0;
        for (auto& e : L->tev) {
            cuda_check(cudaEventSynchronize(e.second), "cudaEventSynchronize");
            float ms = 0.0f;
            cuda_check(cudaEventElapsedTime(&ms, e.first, e.second), "cudaEventElapsedTime");
            tot += ms;
        }
        if (ms_total) *ms_total = tot;
        if (launches) *launches = static_cast<int64_t>(L->tev.size());
    });
}

uint64_t tq_launch_count(const tq_layer* L) { return L ? L->launches.load() : 0; }
void tq_reset_launch_count(tq_layer* L) {
    if (L) L->launches = 0;
}

tq_status tq_route_raw(const float* x, int64_t batch, int64_t in_dim, const float* gate, int64_t num_experts,
                       int64_t top_k, int32_t* ids, float* gates, void* stream) {
    return guarded([&] {
        if (top_k < 1 || top_k > num_experts)
            fail(TQ_ERR_PARAM, "route: top_k " + std::to_string(top_k) + " outside [1, " + std::to_string(num_experts) + "]");
        if (top_k > 64) fail(TQ_ERR_PARAM, "route: GPU router supports top_k <= 64");
        if (batch < 0 || in_dim < 1) fail(TQ_ERR_SHAPE, "route: bad batch / width");
        if (batch == 0) return;
        if (num_experts > 64) fail(TQ_ERR_PARAM, "route: GPU router supports at most 64 experts");
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        DBuf ws, ticket;
        ws.alloc(sizeof(float) * batch * num_experts);
        ticket.alloc(sizeof(int32_t) * batch);
        cuda_check(cudaMemsetAsync(ticket.p, 0, sizeof(int32_t) * batch, st), "cudaMemsetAsync");
        cuda_check(launch_route(x, static_cast<int>(batch), static_cast<int>(in_dim), gate,
                                static_cast<int>(num_experts), static_cast<int>(top_k), 1, 0, 0, ids, gates, nullptr,
                                nullptr, ws.as<float>(), ticket.as<int32_t>(), st),
                   "route_kernel launch");
        cuda_check(cudaStreamSynchronize(st), "stream sync");   // workspace lifetime
    });
}

tq_status tq_route_host(const float* x, int64_t batch, int64_t in_dim, const float* gate, int64_t num_experts,
                        int64_t top_k, int device, int64_t* ids, float* gates) {
    return guarded([&] {
        if (top_k < 1 || top_k > num_experts)
            fail(TQ_ERR_PARAM, "route: top_k " + std::to_string(top_k) + " outside [1, " + std::to_string(num_experts) + "]");
        if (batch < 0 || in_dim < 1) fail(TQ_ERR_SHAPE, "route: bad batch / width");
        if (batch == 0) return;
        cuda_check(cudaSetDevice(device), "cudaSetDevice");
        DBuf xd, gd, idd, gtd;
        xd.alloc(sizeof(float) * batch * in_dim);
        gd.alloc(sizeof(float) * num_experts * in_dim);
        idd.alloc(sizeof(int32_t) * batch * top_k);
        gtd.alloc(sizeof(float) * batch * top_k);
        cuda_check(cudaMemcpy(xd.p, x, sizeof(float) * batch * in_dim, cudaMemcpyHostToDevice), "x H2D");
        cuda_check(cudaMemcpy(gd.p, gate, sizeof(float) * num_experts * in_dim, cudaMemcpyHostToDevice), "gate H2D");
        const tq_status st = tq_route_raw(xd.as<float>(), batch, in_dim, gd.as<float>(), num_experts, top_k,
                                          idd.as<int32_t>(), gtd.as<float>(), nullptr);
        if (st != TQ_OK) fail(st, g_last_error);
        std::vector<int32_t> h(static_cast<size_t>(batch * top_k));
        cuda_check(cudaMemcpy(h.data(), idd.p, sizeof(int32_t) * h.size(), cudaMemcpyDeviceToHost), "ids D2H");
        cuda_check(cudaMemcpy(gates, gtd.p, sizeof(float) * h.size(), cudaMemcpyDeviceToHost), "gates D2H");
        for (size_t t = 0; t < h.size(); ++t) ids[t] = h[t];
    });
}

// ---- expert-parallel stages --------------------------------------------------

int64_t tq_ep_xrow_elems(const tq_layer* L) { return L ? L->g.k_pad : 0; }
int64_t tq_ep_extrow_elems(const tq_layer* L) { return L ? L->g.ext_cols : 0; }

tq_status tq_ep_dispatch_rows(tq_layer* L, const float* x, int64_t batch, const int32_t* ids, const int32_t* perm,
                              uint16_t* xrows, uint16_t* extrows, int path, void* stream) {
    return guarded([&] {
        check_layer(L);
        if (path < 0 || path > 2) fail(TQ_ERR_PARAM, "unknown path " + std::to_string(path));
        if (batch < 0) fail(TQ_ERR_SHAPE, "negative batch");
        if (batch == 0) return;
        if (batch > L->cap) reserve(L, batch);
        cuda_check(cudaSetDevice(L->device), "cudaSetDevice");
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        const Geometry& g = L->g;
        const bool use_lotile = path != TQ_PATH_QMOE;
        const bool use_qmoe = path != TQ_PATH_LOTILE;
        run_route(L, x, batch, false, st);
        const int pns = proj_nsplit(L, batch);
        const LaunchCfg cf = proj_cfg(L, batch);
        PlanArgs pa{};
        pa.ids = ids;
        pa.batch = static_cast<int>(batch);
        pa.top_k = static_cast<int>(g.top_k);
        pa.num_experts = static_cast<int>(g.K);
        pa.e_begin = 0;
        pa.e_end = 0;  // no expert units: this rank only prepares rows
        pa.mb_count = static_cast<int>(g.mb_count);
        pa.kc_total = cf.kc_total;
        pa.nsplit = 1;
        pa.n_ext = cf.n_ext;
        pa.main_kc = 1;
        pa.num_sms = L->num_sms;
        pa.bn = cf.bn;
        pa.proj_mb = use_lotile ? static_cast<int>(L->proj_mb) : 0;
        pa.proj_kc_total = cf.kc_total;
        pa.proj_nsplit = pns;
        pa.perm = L->perm.as<int32_t>();
        pa.inv = L->inv.as<int32_t>();
        pa.offsets = L->offsets.as<int32_t>();
        pa.units = L->units.as<Unit>();
        pa.n_units = L->n_units.as<int32_t>();
        pa.proj_units = L->punits.as<Unit>();
        pa.n_proj_units = L->n_punits.as<int32_t>();
        pa.err_flag = L->err_flag.as<int32_t>();
        cuda_check(launch_plan(pa, st), "plan_kernel launch");
        count_launch(L);
        if (use_lotile && L->proj_mb > 0) {
            GemmParams p = base_params(L, cf, batch);
            p.tmap_x64 = L->map_x16_64;
            p.tmap_e64 = L->map_x16_64;
            p.tmap_x16 = L->map_x16_16;
            p.tmap_e16 = L->map_x16_16;
            p.x_ptr = L->x16.as<__half>();
            p.x_ld = g.k_pad;
            p.e_ptr = L->x16.as<__half>();
            p.e_ld = g.k_pad;
            p.codes = L->pcodes.as<uint8_t>();
            p.weight_stride = L->pweight_stride;
            p.w_outscale = L->p_outscale.as<float>();
            p.units = L->punits.as<Unit>();
            p.n_units = L->n_punits.as<int32_t>();
            p.y = L->zpart.as<float>();
            p.y_split_stride = batch * L->proj_rows;
            p.ldy = static_cast<int32_t>(L->proj_rows);
            p.o_valid = static_cast<int32_t>(L->proj_rows);
            p.o_pad = static_cast<int32_t>(L->proj_o_pad);
            p.bits = kDenseBits;
            const int64_t nunits = L->proj_mb * ((batch + cf.bn - 1) / cf.bn) * pns;
            cuda_check(launch_gemm(p, static_cast<int>(std::min<int64_t>(nunits, L->num_sms)), st),
                       "projection gemm launch");
            count_launch(L);
        }
        GatherArgs ga{};
        ga.x16 = L->x16.as<__half>();
        ga.sx = L->sx.as<float>();
        ga.zpart = L->zpart.as<float>();
        ga.zsplit_stride = batch * L->proj_rows;
        ga.zcols = static_cast<int>(L->proj_rows);
        ga.proj_nsplit = pns;
        ga.ids = ids;
        ga.perm = perm;
        ga.offsets = L->offsets.as<int32_t>();
        ga.pm_of = L->pm_of.as<int32_t>();
        ga.zscale = L->zscale.as<float>();
        ga.rowscale = L->rowscale.as<float>();
        ga.batch = static_cast<int>(batch);
        ga.top_k = static_cast<int>(g.top_k);
        ga.num_experts = static_cast<int>(g.K);
        ga.k_pad = static_cast<int>(g.k_pad);
        ga.groups = static_cast<int>(g.G);
        ga.rank = static_cast<int>(g.r);
        ga.ext_cols = static_cast<int>(g.ext_cols);
        ga.with_shared = 0;
        ga.use_sx = use_qmoe ? 1 : 0;
        ga.use_z = (use_lotile && L->proj_mb > 0) ? 1 : 0;
        ga.xp = reinterpret_cast<__half*>(xrows);
        ga.ep = reinterpret_cast<__half*>(extrows);
        cuda_check(launch_gather(ga, static_cast<int>(batch * g.top_k), st), "gather_kernel launch");
        count_launch(L);
    });
}

tq_status tq_ep_expert_rows(tq_layer* L, const uint16_t* xrows, const uint16_t* extrows, int64_t rows,
                            const int64_t* segments, int64_t nseg, float* yrows, int path, void* stream) {
    return guarded([&] {
        check_layer(L);
        if (path < 0 || path > 2) fail(TQ_ERR_PARAM, "unknown path " + std::to_string(path));
        if (rows < 0 || nseg < 0) fail(TQ_ERR_SHAPE, "negative row / segment count");
        if (rows == 0 || nseg == 0) return;
        cuda_check(cudaSetDevice(L->device), "cudaSetDevice");
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        const Geometry& g = L->g;
        const bool use_qmoe = path != TQ_PATH_LOTILE;
        std::vector<Unit> units;
        const int64_t local = L->e_end - L->e_begin;
        const LaunchCfg cf = cfg64(L);
        int64_t max_tok = 1;
        for (int64_t s = 0; s < nseg; ++s) {
            const int64_t le = segments[3 * s], r0 = segments[3 * s + 1], cnt = segments[3 * s + 2];
            if (le < 0 || le >= local) fail(TQ_ERR_PARAM, "segment expert " + std::to_string(le) + " not resident");
            if (r0 < 0 || cnt < 0 || r0 + cnt > rows) fail(TQ_ERR_SHAPE, "segment rows out of range");
            for (int64_t mb = 0; mb < g.mb_count; ++mb)
                for (int64_t t0 = 0; t0 < cnt; t0 += cf.bn) {
                    Unit u{};
                    u.weight = static_cast<int32_t>(le);
                    u.mb = static_cast<int32_t>(mb);
                    u.x_row = static_cast<int32_t>(r0 + t0);
                    u.n_tok = static_cast<int32_t>(std::min<int64_t>(cf.bn, cnt - t0));
                    max_tok = std::max<int64_t>(max_tok, u.n_tok);
                    u.y_row = u.x_row;
                    u.kc_begin = 0;
                    u.kc_end = static_cast<int16_t>(use_qmoe ? cf.kc_total : 0);
                    u.n_ext = static_cast<int16_t>(cf.n_ext);
                    u.split = 0;
                    units.push_back(u);
                }
        }
        DBuf dunits;
        dunits.alloc(sizeof(Unit) * units.size() + sizeof(int32_t));
        const int32_t nu = static_cast<int32_t>(units.size());
        cuda_check(cudaMemcpyAsync(dunits.p, units.data(), sizeof(Unit) * units.size(), cudaMemcpyHostToDevice, st),
                   "units H2D");
        int32_t* dn = reinterpret_cast<int32_t*>(static_cast<uint8_t*>(dunits.p) + sizeof(Unit) * units.size());
        cuda_check(cudaMemcpyAsync(dn, &nu, sizeof(int32_t), cudaMemcpyHostToDevice, st), "count H2D");
        GemmParams p = base_params(L, cf, max_tok);
        void* xr = const_cast<uint16_t*>(xrows);
        void* er = const_cast<uint16_t*>(extrows);
        p.tmap_x64 = make_map(xr, rows, g.k_pad, 64);
        p.tmap_e64 = make_map(er, rows, g.ext_cols, 64);
        p.tmap_x16 = make_map(xr, rows, g.k_pad, 16);
        p.tmap_e16 = make_map(er, rows, g.ext_cols, 16);
        p.x_ptr = static_cast<const __half*>(xr);
        p.x_ld = g.k_pad;
        p.e_ptr = static_cast<const __half*>(er);
        p.e_ld = g.ext_cols;
        p.codes = L->codes.as<uint8_t>();
        p.weight_stride = L->weight_stride;
        p.scales = L->scales.as<__half>();
        p.ext_blocks = L->ext_blocks.as<uint8_t>();
    p.n_ext64 = static_cast<int32_t>(L->g.n_ext);
        p.w_outscale = L->w_outscale.as<float>();
        p.units = dunits.as<Unit>();
        p.n_units = dn;
        p.y = yrows;
        p.y_split_stride = 0;
        p.ldy = static_cast<int32_t>(g.o);
        p.o_valid = static_cast<int32_t>(g.o);
        p.o_pad = static_cast<int32_t>(g.o_pad);
        p.bits = g.bits;
        p.groups = static_cast<int32_t>(g.G);
        p.rank = static_cast<int32_t>(g.r);
        timed_expert_gemm(L, p, static_cast<int>(std::min<int64_t>(nu, L->num_sms)), st);
        count_launch(L);
        cuda_check(cudaStreamSynchronize(st), "stream sync");  // dunits lifetime
    });
}

tq_status tq_ep_expert_rows_slab(tq_layer* L, const uint16_t* rows, int64_t row_ld, int64_t n_src, int64_t slab,
                                 const int32_t* counts, int64_t e_stride, float* yrows, int path, void* stream) {
    return guarded([&] {
        check_layer(L);
        if (path < 0 || path > 2) fail(TQ_ERR_PARAM, "unknown path " + std::to_string(path));
        const Geometry& g = L->g;
        const int64_t local = L->e_end - L->e_begin;
        if (n_src < 1 || slab < 0 || e_stride < local) fail(TQ_ERR_SHAPE, "slab layout: bad source count / capacity / stride");
        if (row_ld < g.k_pad + g.ext_cols || (row_ld % 8) != 0)
            fail(TQ_ERR_SHAPE, "slab rows hold [x (" + std::to_string(g.k_pad) + ") | ext (" +
                                   std::to_string(g.ext_cols) + ")] fp16, 16-byte aligned");
        if (n_src * local > 1024) fail(TQ_ERR_PARAM, "slab layout: at most 1024 (source, expert) segments");
        if (slab == 0 || local == 0) return;
        cuda_check(cudaSetDevice(L->device), "cudaSetDevice");
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        const LaunchCfg cf = cfg64(L);
        // units on the device: capacity for the worst split of slab rows over the experts
        const int64_t cap = n_src * (local * g.mb_count + g.mb_count * ((slab + cf.bn - 1) / cf.bn));
        if (cap > L->ep_units_cap) {
            L->ep_units.alloc(sizeof(Unit) * cap);
            L->ep_nunits.alloc(sizeof(int32_t));
            L->ep_units_cap = cap;
        }
        const bool use_qmoe = path != TQ_PATH_LOTILE;
        cuda_check(launch_ep_units(counts, static_cast<int>(n_src), static_cast<int>(e_stride), static_cast<int>(local),
                                   static_cast<int>(slab), static_cast<int>(g.mb_count), cf.bn,
                                   use_qmoe ? cf.kc_total : 0, cf.n_ext, L->ep_units.as<Unit>(),
                                   L->ep_nunits.as<int32_t>(), st),
                   "ep units");
        count_launch(L);
        const int64_t nrows = n_src * slab;
        GemmParams p = base_params(L, cf, cf.bn);
        void* xr = const_cast<uint16_t*>(rows);
        void* er = const_cast<uint16_t*>(rows + g.k_pad);
        p.tmap_x64 = make_map(xr, nrows, g.k_pad, 64, row_ld);
        p.tmap_e64 = make_map(er, nrows, g.ext_cols, 64, row_ld);
        p.tmap_x16 = make_map(xr, nrows, g.k_pad, 16, row_ld);
        p.tmap_e16 = make_map(er, nrows, g.ext_cols, 16, row_ld);
        p.x_ptr = static_cast<const __half*>(xr);
        p.x_ld = row_ld;
        p.e_ptr = static_cast<const __half*>(er);
        p.e_ld = row_ld;
        p.codes = L->codes.as<uint8_t>();
        p.weight_stride = L->weight_stride;
        p.scales = L->scales.as<__half>();
        p.ext_blocks = L->ext_blocks.as<uint8_t>();
        p.n_ext64 = static_cast<int32_t>(g.n_ext);
        p.w_outscale = L->w_outscale.as<float>();
        p.units = L->ep_units.as<Unit>();
        p.n_units = L->ep_nunits.as<int32_t>();
        p.y = yrows;
        p.y_split_stride = 0;
        p.ldy = static_cast<int32_t>(g.o);
        p.o_valid = static_cast<int32_t>(g.o);
        p.o_pad = static_cast<int32_t>(g.o_pad);
        p.bits = g.bits;
        p.groups = static_cast<int32_t>(g.G);
        p.rank = static_cast<int32_t>(g.r);
        timed_expert_gemm(L, p, L->num_sms, st);
        count_launch(L);
    });
}

tq_status tq_ep_combine(tq_layer* L, const float* x, int64_t batch, const float* yrows, const int32_t* inv,
                        const float* gates, float* y, int path, void* stream) {
    return guarded([&] {
        check_layer(L);
        if (path < 0 || path > 2) fail(TQ_ERR_PARAM, "unknown path " + std::to_string(path));
        if (batch < 0) fail(TQ_ERR_SHAPE, "negative batch");
        if (batch == 0) return;
        if (batch > L->cap) reserve(L, batch);
        cuda_check(cudaSetDevice(L->device), "cudaSetDevice");
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        const Geometry& g = L->g;
        const bool shared = path != TQ_PATH_LOTILE && g.S > 0;
        if (shared) {
            // shared experts on the home tokens: rows 0..B-1 of xperm, outputs s*B + b of ypart
            run_route(L, x, batch, false, st);
            GatherArgs ga{};
            ga.x16 = L->x16.as<__half>();
            ga.sx = L->sx.as<float>();
            ga.zpart = L->zpart.as<float>();
            ga.offsets = L->offsets.as<int32_t>();  // offsets[0] == 0: no routed rows
            ga.pm_of = L->pm_of.as<int32_t>();
            ga.zscale = L->zscale.as<float>();
            ga.rowscale = L->rowscale.as<float>();
            ga.batch = static_cast<int>(batch);
            ga.top_k = static_cast<int>(g.top_k);
            ga.num_experts = 0;
            ga.k_pad = static_cast<int>(g.k_pad);
            ga.groups = static_cast<int>(g.G);
            ga.rank = static_cast<int>(g.r);
            ga.ext_cols = static_cast<int>(g.ext_cols);
            ga.with_shared = 1;
            ga.use_sx = 1;
            ga.use_z = 0;
            ga.xp = L->xperm.as<__half>();
            ga.ep = L->extperm.as<__half>();
            cuda_check(launch_gather(ga, static_cast<int>(batch), st), "gather_kernel launch");
            count_launch(L);
            std::vector<Unit> units;
            const int64_t local = L->e_end - L->e_begin;
            const LaunchCfg cf = cfg64(L);
            for (int64_t s = 0; s < g.S; ++s)
                for (int64_t mb = 0; mb < g.mb_count; ++mb)
                    for (int64_t t0 = 0; t0 < batch; t0 += cf.bn) {
                        Unit u{};
                        u.weight = static_cast<int32_t>(local + s);
                        u.mb = static_cast<int32_t>(mb);
                        u.x_row = static_cast<int32_t>(t0);
                        u.n_tok = static_cast<int32_t>(std::min<int64_t>(cf.bn, batch - t0));
                        u.y_row = static_cast<int32_t>(s * batch + t0);
                        u.kc_begin = 0;
                        u.kc_end = static_cast<int16_t>(cf.kc_total);
                        u.n_ext = static_cast<int16_t>(cf.n_ext);
                        units.push_back(u);
                    }
            const int32_t nu = static_cast<int32_t>(units.size());
            cuda_check(cudaMemcpyAsync(L->units.p, units.data(), sizeof(Unit) * units.size(), cudaMemcpyHostToDevice, st),
                       "units H2D");
            cuda_check(cudaMemcpyAsync(L->n_units.p, &nu, sizeof(int32_t), cudaMemcpyHostToDevice, st), "count H2D");
            GemmParams p = base_params(L, cf, batch);
            p.tmap_x64 = L->map_xp64;
            p.tmap_e64 = L->map_ep64;
            p.tmap_x16 = L->map_xp16;
            p.tmap_e16 = L->map_ep16;
            p.x_ptr = L->xperm.as<__half>();
            p.x_ld = g.k_pad;
            p.e_ptr = L->extperm.as<__half>();
            p.e_ld = g.ext_cols;
            p.codes = L->codes.as<uint8_t>();
            p.weight_stride = L->weight_stride;
            p.scales = L->scales.as<__half>();
            p.ext_blocks = L->ext_blocks.as<uint8_t>();
    p.n_ext64 = static_cast<int32_t>(L->g.n_ext);
            p.w_outscale = L->w_outscale.as<float>();
            p.units = L->units.as<Unit>();
            p.n_units = L->n_units.as<int32_t>();
            p.y = L->ypart.as<float>();
            p.ldy = static_cast<int32_t>(g.o);
            p.o_valid = static_cast<int32_t>(g.o);
            p.o_pad = static_cast<int32_t>(g.o_pad);
            p.bits = g.bits;
            p.groups = static_cast<int32_t>(g.G);
            p.rank = static_cast<int32_t>(g.r);
            cuda_check(launch_gemm(p, static_cast<int>(std::min<int64_t>(nu, L->num_sms)), st), "shared gemm launch");
            count_launch(L);
            cuda_check(cudaStreamSynchronize(st), "stream sync");  // host unit table lifetime
        }
        CombineArgs ca{};
        ca.y = yrows;
        ca.split_stride = 0;
        ca.nsplit = 1;
        ca.inv = inv;
        ca.gates = gates;
        ca.offsets = nullptr;
        ca.num_experts = static_cast<int>(g.K);
        ca.batch = static_cast<int>(batch);
        ca.top_k = static_cast<int>(g.top_k);
        ca.out_dim = static_cast<int>(g.o);
        ca.num_shared = shared ? static_cast<int>(g.S) : 0;
        ca.use_routed = 1;
        ca.ysh = L->ypart.as<float>();
        ca.sh_split_stride = 0;
        ca.sh_nsplit = 1;
        ca.sh_from_offsets = 0;
        ca.out = y;
        cuda_check(launch_combine(ca, st), "combine_kernel launch");
        count_launch(L);
    });
}

}  // extern "C"

// ---------------------------------------------------------------------------
// artifact producer hot spots: estimate_hessian, spd_inverse,
// quantize_rtn, quantize_gptq, proxy_loss (quant.cpp:72-221,325-343) on device
// arrays.  Bit-identical to the reference (tq_producer.cu).
// ---------------------------------------------------------------------------

namespace {

// stream-ordered device scratch
struct AsyncBuf {
    void* p = nullptr;
    cudaStream_t s = nullptr;
    AsyncBuf(size_t bytes, cudaStream_t st) : s(st) {
        if (bytes) cuda_check(cudaMallocAsync(&p, bytes, st), "cudaMallocAsync (producer scratch)");
    }
    ~AsyncBuf() {
        if (p) cudaFreeAsync(p, s);
    }
    AsyncBuf(const AsyncBuf&) = delete;
    AsyncBuf& operator=(const AsyncBuf&) = delete;
    template <class T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

void check_quant_bits(int bits) {
    if (bits != 2 && bits != 3 && bits != 4 && bits != 8)
        fail(TQ_ERR_PARAM, "quantizer bits must be in {2,3,4,8}, got " + std::to_string(bits));
}

// spd_inverse into hinv (n x n f64, device); NumericError as quant.cpp:80-85
void spd_inverse_dev(const float* h, int64_t n, double* hinv, cudaStream_t st) {
    if (n == 0) return;
    AsyncBuf chol(sizeof(double) * n * n, st), linv(sizeof(double) * n * n, st), status(spd_status_bytes(), st);
    cuda_check(launch_spd_inverse(h, n, chol.as<double>(), linv.as<double>(), hinv, status.p, st),
               "spd_inverse launch");
    std::vector<unsigned char> host(spd_status_bytes());
    cuda_check(cudaMemcpyAsync(host.data(), status.p, host.size(), cudaMemcpyDeviceToHost, st), "spd status D2H");
    cuda_check(cudaStreamSynchronize(st), "stream sync");
    int failed = 0;
    int64_t col = 0;
    double pivot = 0.0;
    spd_status_read(host.data(), &failed, &col, &pivot);
    if (failed)
        fail(TQ_ERR_NUMERIC, "Hessian is singular after damping (pivot " + std::to_string(pivot) + " at column " +
                                 std::to_string(col) + "); increase damping_fraction");
}

double proxy_loss_dev(const float* original, int64_t rows, int64_t cols, const uint8_t* codes, const float* scales,
                      const int32_t* zeros, int64_t gs, const float* h, cudaStream_t st) {
    if (rows == 0 || cols == 0) return 0.0;
    const int64_t chunk = std::min<int64_t>(rows, std::max<int64_t>(64, (int64_t{256} << 20) / (8 * cols)));
    AsyncBuf he(sizeof(double) * chunk * cols, st), rowsum(sizeof(double) * rows, st), total(sizeof(double), st);
    cuda_check(launch_proxy_loss(original, codes, scales, zeros, rows, cols, gs, h, chunk, he.as<double>(),
                                 rowsum.as<double>(), total.as<double>(), st),
               "proxy_loss launch");
    double out = 0.0;
    cuda_check(cudaMemcpyAsync(&out, total.p, sizeof(double), cudaMemcpyDeviceToHost, st), "proxy D2H");
    cuda_check(cudaStreamSynchronize(st), "stream sync");
    return out;
}

}  // namespace

extern "C" {

tq_status tq_estimate_hessian(const float* calib, int64_t tokens, int64_t dim, double damping_fraction, float* h,
                              double* damping_out, void* stream) {
    return guarded([&] {
        if (tokens < 0 || dim < 0) fail(TQ_ERR_PARAM, "estimate_hessian: negative size");
        if (tokens == 0 || dim == 0) fail(TQ_ERR_DATA, "estimate_hessian: empty calibration set");
        if (damping_fraction < 0.0) fail(TQ_ERR_PARAM, "estimate_hessian: damping_fraction must be >= 0");
        if (!calib || !h) fail(TQ_ERR_PARAM, "estimate_hessian: null buffer");
        const cudaStream_t st = static_cast<cudaStream_t>(stream);
        AsyncBuf acc(sizeof(double) * dim * dim, st), lam(sizeof(double), st);
        cuda_check(launch_estimate_hessian(calib, tokens, dim, damping_fraction, acc.as<double>(), lam.as<double>(),
                                           h, st),
                   "estimate_hessian launch");
        if (damping_out) {
            cuda_check(cudaMemcpyAsync(damping_out, lam.p, sizeof(double), cudaMemcpyDeviceToHost, st), "lambda D2H");
            cuda_check(cudaStreamSynchronize(st), "stream sync");
        }
    });
}

tq_status tq_spd_inverse(const float* h, int64_t n, double* hinv, void* stream) {
    return guarded([&] {
        if (n < 0 || (n > 0 && (!h || !hinv))) fail(TQ_ERR_PARAM, "spd_inverse: bad arguments");
        spd_inverse_dev(h, n, hinv, static_cast<cudaStream_t>(stream));
    });
}

tq_status tq_quantize_rtn(const float* r, int64_t rows, int64_t cols, int bits, int64_t group_size, uint8_t* codes,
                          float* scales, int32_t* zeros, void* stream) {
    return guarded([&] {
        check_quant_bits(bits);
        if (group_size < 1) fail(TQ_ERR_PARAM, "quantize_rtn: group_size must be >= 1");
        if (rows <= 0 || cols <= 0) fail(TQ_ERR_PARAM, "quantize_rtn: empty input");
        if (!r || !codes || !scales || !zeros) fail(TQ_ERR_PARAM, "quantize_rtn: null buffer");
        const cudaStream_t st = static_cast<cudaStream_t>(stream);
        cuda_check(launch_make_grids(r, rows, cols, bits, group_size, scales, zeros, st), "grids launch");
        cuda_check(launch_rtn_codes(r, rows, cols, bits, group_size, scales, zeros, codes, st), "rtn launch");
    });
}

tq_status tq_quantize_gptq(const float* r, int64_t rows, int64_t cols, const float* h, int bits, int64_t group_size,
                           uint8_t* codes, float* scales, int32_t* zeros, int32_t* used_rtn, void* stream) {
    return guarded([&] {
        check_quant_bits(bits);
        if (group_size < 1) fail(TQ_ERR_PARAM, "quantize_gptq: group_size must be >= 1");
        if (rows < 0 || cols < 0) fail(TQ_ERR_PARAM, "quantize_gptq: negative size");
        if (cols > 0 && gptq_rows_per_cta(cols, group_size) == 0)
            fail(TQ_ERR_PARAM, "quantize_gptq: in_dim " + std::to_string(cols) +
                                   " exceeds the engine's limit (one working row and its grids in shared memory)");
        const cudaStream_t st = static_cast<cudaStream_t>(stream);
        AsyncBuf hinv(sizeof(double) * cols * cols, st);
        spd_inverse_dev(h, cols, hinv.as<double>(), st);                       // quant.cpp:187
        if (rows == 0 || cols == 0) fail(TQ_ERR_PARAM, "quantize_rtn: empty input");   // quant.cpp:218 -> :155
        if (!r || !codes || !scales || !zeros) fail(TQ_ERR_PARAM, "quantize_gptq: null buffer");
        cuda_check(launch_make_grids(r, rows, cols, bits, group_size, scales, zeros, st), "grids launch");
        cuda_check(launch_gptq(r, rows, cols, bits, group_size, scales, zeros, hinv.as<double>(), codes, st),
                   "gptq launch");
        // keep the better of GPTQ and plain rounding (same grids) -- quant.cpp:216-219
        AsyncBuf rtn(static_cast<size_t>(rows * cols), st);
        cuda_check(launch_rtn_codes(r, rows, cols, bits, group_size, scales, zeros, rtn.as<uint8_t>(), st),
                   "rtn launch");
        const double lg = proxy_loss_dev(r, rows, cols, codes, scales, zeros, group_size, h, st);
        const double lr = proxy_loss_dev(r, rows, cols, rtn.as<uint8_t>(), scales, zeros, group_size, h, st);
        const bool take_rtn = lg > lr;
        if (take_rtn)
            cuda_check(cudaMemcpyAsync(codes, rtn.p, static_cast<size_t>(rows * cols), cudaMemcpyDeviceToDevice, st),
                       "rtn codes D2D");
        if (used_rtn) *used_rtn = take_rtn ? 1 : 0;
    });
}

tq_status tq_proxy_loss(const float* original, int64_t rows, int64_t cols, const uint8_t* codes, const float* scales,
                        const int32_t* zeros, int bits, int64_t group_size, const float* h, double* loss,
                        void* stream) {
    return guarded([&] {
        check_quant_bits(bits);
        if (group_size < 1) fail(TQ_ERR_PARAM, "proxy_loss: group_size must be >= 1");
        if (rows < 0 || cols < 0 || !loss) fail(TQ_ERR_PARAM, "proxy_loss: bad arguments");
        *loss = proxy_loss_dev(original, rows, cols, codes, scales, zeros, group_size, h,
                               static_cast<cudaStream_t>(stream));
    });
}

}  // extern "C"

// ---------------------------------------------------------------------------
// sketch_lowrank (lowrank.cpp:194-247) with the mat-vecs on the device
// ---------------------------------------------------------------------------

namespace {

// The reference's counter-based generator (rng.hpp: splitmix64 finalizer over
// seed + n * golden gamma, Box-Muller with a cached spare), restated: the probes
// are drawn here on the host with the host's libm, exactly as the reference
// draws them, and uploaded.
class SketchRng {
public:
    explicit SketchRng(uint64_t seed) : seed_(seed) {}
    double gaussian() {
        if (spare_ok_) {
            spare_ok_ = false;
            return spare_;
        }
        const double u1 = 1.0 - unit();
        const double u2 = unit();
        const double radius = std::sqrt(-2.0 * std::log(u1));
        const double angle = 6.283185307179586476925286766559 * u2;
        spare_ = radius * std::sin(angle);
        spare_ok_ = true;
        return radius * std::cos(angle);
    }

private:
    static uint64_t mix(uint64_t z) {
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        return z ^ (z >> 31);
    }
    double unit() { return static_cast<double>(mix(seed_ + (++counter_) * 0x9E3779B97F4A7C15ull) >> 11) * 0x1.0p-53; }
    uint64_t seed_;
    uint64_t counter_ = 0;
    double spare_ = 0.0;
    bool spare_ok_ = false;
};

double read_scalar(const double* d, cudaStream_t st) {
    double v = 0.0;
    cuda_check(cudaMemcpyAsync(&v, d, sizeof(double), cudaMemcpyDeviceToHost, st), "scalar D2H");
    cuda_check(cudaStreamSynchronize(st), "stream sync");
    return v;
}

}  // namespace

extern "C" tq_status tq_sketch_lowrank(const float* w, int64_t rows, int64_t cols, int64_t rank, int power_iters,
                                       uint64_t seed, float* left, float* right, float* singulars, void* stream) {
    return guarded([&] {
        if (rows <= 0 || cols <= 0) fail(TQ_ERR_PARAM, "sketch_lowrank: input matrix is empty");
        const int64_t cap = std::min(rows, cols);
        if (rank < 1 || rank > cap)
            fail(TQ_ERR_PARAM, "sketch_lowrank: rank " + std::to_string(rank) + " outside [1, " + std::to_string(cap) +
                                   "] for a " + std::to_string(rows) + "x" + std::to_string(cols) + " matrix");
        if (power_iters < 0) fail(TQ_ERR_PARAM, "sketch_lowrank: power_iters must be >= 0");
        if (!w || !left || !right || !singulars) fail(TQ_ERR_PARAM, "sketch_lowrank: null buffer");
        const cudaStream_t st = static_cast<cudaStream_t>(stream);
        AsyncBuf work(sizeof(double) * rows * cols, st), q(sizeof(double) * rows, st), t(sizeof(double) * cols, st),
            us(sizeof(double) * rank * rows, st), vs(sizeof(double) * rank * cols, st), sig(sizeof(double) * rank, st),
            nrm(sizeof(double), st), order_d(sizeof(int32_t) * rank, st);
        cuda_check(launch_widen(w, rows * cols, work.as<double>(), st), "widen launch");
        SketchRng rng(seed);
        std::vector<double> probe(static_cast<size_t>(cols)), sigmas(static_cast<size_t>(rank), 0.0);
        double* W = work.as<double>();
        double* Q = q.as<double>();
        double* T = t.as<double>();
        for (int64_t j = 0; j < rank; ++j) {
            for (double& p : probe) p = rng.gaussian();
            cuda_check(cudaMemcpyAsync(T, probe.data(), sizeof(double) * cols, cudaMemcpyHostToDevice, st),
                       "probe H2D");
            cuda_check(launch_matvec(W, rows, cols, T, Q, st), "matvec launch");
            cuda_check(launch_norm2(Q, rows, nrm.as<double>(), st), "norm launch");
            bool dead = read_scalar(nrm.as<double>(), st) == 0.0;   // (also orders the probe buffer's reuse)
            if (!dead) {
                cuda_check(launch_div_by(Q, rows, nrm.as<double>(), Q, st), "scale launch");
                for (int it = 0; it < power_iters && !dead; ++it) {
                    cuda_check(launch_mattvec(W, rows, cols, Q, T, st), "mattvec launch");
                    cuda_check(launch_matvec(W, rows, cols, T, Q, st), "matvec launch");
                    cuda_check(launch_norm2(Q, rows, nrm.as<double>(), st), "norm launch");
                    if (read_scalar(nrm.as<double>(), st) == 0.0) dead = true;
                    else cuda_check(launch_div_by(Q, rows, nrm.as<double>(), Q, st), "scale launch");
                }
            }
            double* Uj = us.as<double>() + j * rows;
            double* Vj = vs.as<double>() + j * cols;
            if (!dead) {
                cuda_check(launch_mattvec(W, rows, cols, Q, T, st), "mattvec launch");
                double* Sj = sig.as<double>() + j;
                cuda_check(launch_norm2(T, cols, Sj, st), "norm launch");
                const double sigma = read_scalar(Sj, st);
                if (sigma == 0.0) {
                    dead = true;
                } else {
                    sigmas[static_cast<size_t>(j)] = sigma;
                    cuda_check(cudaMemcpyAsync(Uj, Q, sizeof(double) * rows, cudaMemcpyDeviceToDevice, st), "u D2D");
                    cuda_check(launch_div_by(T, cols, Sj, Vj, st), "v launch");
                    cuda_check(launch_deflate(W, rows, cols, Sj, Uj, Vj, st), "deflate launch");
                }
            }
            if (dead) {   // basis_triple (lowrank.cpp:101-108)
                cuda_check(cudaMemsetAsync(Uj, 0, sizeof(double) * rows, st), "u memset");
                cuda_check(cudaMemsetAsync(Vj, 0, sizeof(double) * cols, st), "v memset");
                const double one = 1.0;
                cuda_check(cudaMemcpyAsync(Uj + j % rows, &one, sizeof(double), cudaMemcpyHostToDevice, st), "u e_j");
                cuda_check(cudaMemcpyAsync(Vj + j % cols, &one, sizeof(double), cudaMemcpyHostToDevice, st), "v e_j");
                cuda_check(cudaStreamSynchronize(st), "stream sync");   // (&one is a stack value)
                sigmas[static_cast<size_t>(j)] = 0.0;
            }
        }
        // nonincreasing sigma, stable (lowrank.cpp:80-82)
        std::vector<int32_t> order(static_cast<size_t>(rank));
        for (int64_t j = 0; j < rank; ++j) order[static_cast<size_t>(j)] = static_cast<int32_t>(j);
        std::stable_sort(order.begin(), order.end(),
                         [&](int32_t a, int32_t b) { return sigmas[static_cast<size_t>(a)] > sigmas[static_cast<size_t>(b)]; });
        std::vector<float> sv(static_cast<size_t>(rank));
        for (int64_t p2 = 0; p2 < rank; ++p2) sv[static_cast<size_t>(p2)] = static_cast<float>(sigmas[order[static_cast<size_t>(p2)]]);
        cuda_check(cudaMemcpyAsync(order_d.p, order.data(), sizeof(int32_t) * rank, cudaMemcpyHostToDevice, st),
                   "order H2D");
        cuda_check(cudaMemcpyAsync(singulars, sv.data(), sizeof(float) * rank, cudaMemcpyHostToDevice, st),
                   "singulars H2D");
        cuda_check(launch_pack_triples(us.as<double>(), vs.as<double>(), order_d.as<int32_t>(), rank, rows, cols, left,
                                       right, st),
                   "pack launch");
        cuda_check(cudaStreamSynchronize(st), "stream sync");   // host order / sv lifetimes
    });
}
