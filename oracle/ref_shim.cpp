// TEST INFRASTRUCTURE ONLY -- never linked into or called by the product path.
//
// extern "C" veneer over the UNMODIFIED reference library compiled from
// /root/reference/proj/src (see oracle/Makefile).  It lets the pytest suite,
// __graft_entry__.smoke() and bench.py's cpu_baseline leg drive the
// reference's own code path through ctypes:
//
//   * tq_ref_load / tq_ref_forward : read_artifact (io.cpp:679) + route
//     (moe.cpp:43) + tileq_forward (infer.cpp:182), i.e. exactly what the
//     reference Python binding forward_from_artifact does
//     (bindings/py_module.cpp:112-117), plus the two halves qmoe_forward
//     (infer.cpp:40) and lotile_forward (infer.cpp:53) separately.
//   * tq_ref_route  : route() on raw arrays (moe.cpp:43-89).
//   * tq_ref_unpack : unpack_codes() (codec.cpp:168-195).
//   * tq_ref_make_artifact : the artifact factory.  It runs the stage
//     sequence of quantize_moe (pipeline.cpp:138-230) with the same stage
//     seeds but skips proxy_loss (quant.cpp:325-343), which only feeds the
//     report; the artifact bytes are unchanged (checked by
//     tests/test_cpu_oracle.py::test_factory_stage_replay_matches_quantize_moe
//     against quantize_moe itself on a small shape).
//     Inputs follow the CLI synth command (tileq_main.cpp:356-410):
//     synth_experts + gaussian gate from derive(seed, 6) + calibration
//     tokens from derive(seed, 5) (signs -> folded descale tier, gaussians ->
//     general tier).
//
//   * tq_ref_estimate_hessian / tq_ref_quantize / tq_ref_proxy_loss: the
//     artifact producer's hot spots (quant.cpp:116-221,325-343) on raw arrays.
//
// Errors never cross this boundary as exceptions: every entry returns 0 on
// success or a tileq error class code and writes the message to errbuf.

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "tileq/codec.hpp"
#include "tileq/errors.hpp"
#include "tileq/infer.hpp"
#include "tileq/io.hpp"
#include "tileq/lowrank.hpp"
#include "tileq/moe.hpp"
#include "tileq/pipeline.hpp"
#include "tileq/quant.hpp"
#include "tileq/rng.hpp"
#include "tileq/tiler.hpp"

using namespace tileq;

namespace {

int classify(const std::exception& e) {
    if (dynamic_cast<const ShapeError*>(&e)) return 1;
    if (dynamic_cast<const ParamError*>(&e)) return 2;
    if (dynamic_cast<const SizeError*>(&e)) return 3;
    if (dynamic_cast<const FormatError*>(&e)) return 4;
    if (dynamic_cast<const IoError*>(&e)) return 5;
    if (dynamic_cast<const NumericError*>(&e)) return 6;
    if (dynamic_cast<const DataError*>(&e)) return 7;
    return 99;
}

void put_err(char* buf, int len, const char* msg) {
    if (buf == nullptr || len <= 0) return;
    std::strncpy(buf, msg, static_cast<std::size_t>(len - 1));
    buf[len - 1] = '\0';
}

template <class F>
int guarded(char* errbuf, int errlen, F&& body) {
    try {
        body();
        return 0;
    } catch (const std::exception& e) {
        put_err(errbuf, errlen, e.what());
        return classify(e);
    }
}

DenseMatrix wrap(const float* data, std::int64_t rows, std::int64_t cols) {
    DenseMatrix m(static_cast<std::size_t>(rows), static_cast<std::size_t>(cols));
    if (!m.data.empty()) std::memcpy(m.data.data(), data, m.data.size() * sizeof(float));
    return m;
}

void copy_out(const DenseMatrix& m, float* dst) {
    if (!m.data.empty()) std::memcpy(dst, m.data.data(), m.data.size() * sizeof(float));
}

struct RefHandle {
    LoadedArtifact art;
};

// pipeline.cpp:20-24 stage streams.
constexpr std::uint64_t kFeatureStream = 1;
constexpr std::uint64_t kClusterStream = 2;
constexpr std::uint64_t kDecomposeStream = 3;
// tileq_main.cpp:46-47 CLI synth streams.
constexpr std::uint64_t kCalibStream = 5;
constexpr std::uint64_t kGateStream = 6;

} // namespace

extern "C" {

int tq_ref_load(const char* dir, int verify_crc, void** out, char* errbuf, int errlen) {
    return guarded(errbuf, errlen, [&] {
        auto* h = new RefHandle{read_artifact(dir, verify_crc != 0)};
        *out = h;
    });
}

void tq_ref_free(void* h) { delete static_cast<RefHandle*>(h); }

int tq_ref_spec(void* hv, std::int64_t* out6) {
    auto* h = static_cast<RefHandle*>(hv);
    const MoELayerSpec& s = h->art.layer.spec;
    out6[0] = static_cast<std::int64_t>(s.num_experts);
    out6[1] = static_cast<std::int64_t>(s.top_k);
    out6[2] = static_cast<std::int64_t>(s.in_dim);
    out6[3] = static_cast<std::int64_t>(s.out_dim);
    out6[4] = static_cast<std::int64_t>(s.num_shared);
    out6[5] = static_cast<std::int64_t>(h->art.layer.tiled.rank);
    return 0;
}

// mode: 0 = tileq_forward (qmoe + lotile), 1 = qmoe_forward, 2 = lotile_forward.
// threads > 1 token-shards the batch: each worker runs route + forward on a
// contiguous row slice (rows are independent), output-identical.
int tq_ref_forward(void* hv, const float* x, std::int64_t batch, int mode, int threads,
                   float* y, std::int64_t* ids, float* gates, char* errbuf, int errlen) {
    auto* h = static_cast<RefHandle*>(hv);
    const TileQLayer& layer = h->art.layer;
    const std::int64_t in_dim = static_cast<std::int64_t>(layer.spec.in_dim);
    const std::int64_t out_dim = static_cast<std::int64_t>(layer.spec.out_dim);
    const std::int64_t top_k = static_cast<std::int64_t>(layer.spec.top_k);
    auto run_slice = [&](std::int64_t b0, std::int64_t b1) {
        DenseMatrix xm = wrap(x + b0 * in_dim, b1 - b0, in_dim);
        RoutingDecision routing = route(xm, layer.gate_weights, layer.spec.top_k);
        DenseMatrix out;
        if (mode == 1) out = qmoe_forward(xm, layer, routing);
        else if (mode == 2) out = lotile_forward(xm, layer.tiled, routing);
        else out = tileq_forward(xm, layer, routing);
        std::memcpy(y + b0 * out_dim, out.data.data(), out.data.size() * sizeof(float));
        for (std::int64_t b = 0; b < b1 - b0; ++b)
            for (std::int64_t t = 0; t < top_k; ++t) {
                if (ids) ids[(b0 + b) * top_k + t] = static_cast<std::int64_t>(routing.id_at(b, t));
                if (gates) gates[(b0 + b) * top_k + t] = routing.gate_at(b, t);
            }
    };
    return guarded(errbuf, errlen, [&] {
        if (threads <= 1 || batch <= 1) {
            run_slice(0, batch);
            return;
        }
        const std::int64_t nw = std::min<std::int64_t>(threads, batch);
        std::vector<std::thread> pool;
        std::vector<std::string> errs(static_cast<std::size_t>(nw));
        for (std::int64_t w = 0; w < nw; ++w) {
            const std::int64_t b0 = batch * w / nw, b1 = batch * (w + 1) / nw;
            pool.emplace_back([&, w, b0, b1] {
                try {
                    run_slice(b0, b1);
                } catch (const std::exception& e) {
                    errs[static_cast<std::size_t>(w)] = e.what();
                }
            });
        }
        for (auto& t : pool) t.join();
        for (auto& e : errs)
            if (!e.empty()) throw Error(e);
    });
}

int tq_ref_route(const float* x, std::int64_t batch, std::int64_t in_dim, const float* gate,
                 std::int64_t num_experts, std::int64_t top_k, std::int64_t* ids, float* gates,
                 char* errbuf, int errlen) {
    return guarded(errbuf, errlen, [&] {
        DenseMatrix xm = wrap(x, batch, in_dim);
        DenseMatrix gm = wrap(gate, num_experts, in_dim);
        RoutingDecision r = route(xm, gm, static_cast<std::size_t>(top_k));
        for (std::size_t f = 0; f < r.expert_ids.size(); ++f) ids[f] = static_cast<std::int64_t>(r.expert_ids[f]);
        copy_out(r.gates, gates);
    });
}

int tq_ref_unpack(const std::uint8_t* bytes, std::int64_t nbytes, int bits, std::int64_t count,
                  std::uint32_t* out, char* errbuf, int errlen) {
    return guarded(errbuf, errlen, [&] {
        std::vector<std::uint8_t> v(bytes, bytes + nbytes);
        std::vector<std::uint32_t> c = unpack_codes(v, bits, static_cast<std::size_t>(count));
        std::memcpy(out, c.data(), c.size() * sizeof(std::uint32_t));
    });
}

int tq_ref_pack(const std::uint32_t* codes, std::int64_t count, int bits, std::uint8_t* out,
                char* errbuf, int errlen) {
    return guarded(errbuf, errlen, [&] {
        std::vector<std::uint32_t> v(codes, codes + count);
        std::vector<std::uint8_t> b = pack_codes(v, bits);
        std::memcpy(out, b.data(), b.size());
    });
}

int tq_ref_f16_to_f32(const std::uint16_t* bits, std::int64_t n, float* out) {
    for (std::int64_t t = 0; t < n; ++t) out[t] = half_bits_to_float(bits[t]);
    return 0;
}

int tq_ref_f32_to_f16(const float* v, std::int64_t n, std::uint16_t* out) {
    for (std::int64_t t = 0; t < n; ++t) out[t] = float_to_half_bits(v[t]);
    return 0;
}

// Dequantized residual of routed expert e (or shared expert e - K when
// e >= K) exactly as dequantize() (quant.cpp:285-323) produces it.
int tq_ref_dequantize(void* hv, std::int64_t e, float* out, char* errbuf, int errlen) {
    auto* h = static_cast<RefHandle*>(hv);
    return guarded(errbuf, errlen, [&] {
        const TileQLayer& L = h->art.layer;
        const std::size_t k = static_cast<std::size_t>(e);
        const QuantizedExpert& q =
            k < L.quantized.size() ? L.quantized[k] : L.shared_quantized.at(k - L.quantized.size());
        copy_out(dequantize(q), out);
    });
}

// reconstruct_expert (tiler.cpp:337-358) of routed expert e.
int tq_ref_reconstruct(void* hv, std::int64_t e, float* out, char* errbuf, int errlen) {
    auto* h = static_cast<RefHandle*>(hv);
    return guarded(errbuf, errlen, [&] {
        copy_out(reconstruct_expert(h->art.layer.tiled, static_cast<std::size_t>(e)), out);
    });
}

// Artifact factory (see header comment).  calib_kind: 0 = random signs
// (neutral scaling, folded tier), 1 = gaussian (general tier), 2 = empty
// (all-ones scaling).  full_pipeline != 0 calls quantize_moe itself
// (including proxy_loss) for cross-checking the stage replay.
int tq_ref_make_artifact(const char* dir, std::int64_t num_experts, std::int64_t top_k,
                         std::int64_t in_dim, std::int64_t out_dim, std::int64_t num_shared,
                         std::int64_t grid_rows, std::int64_t grid_cols, std::int64_t rank,
                         int bits, std::int64_t group_size, int calib_kind,
                         std::int64_t calib_tokens, double noise, double mix_scale,
                         std::int64_t planted_rank, std::uint64_t seed, int full_pipeline,
                         int quantizer, std::int64_t sub_dim, char* errbuf, int errlen) {
    return guarded(errbuf, errlen, [&] {
        MoELayerSpec spec{static_cast<std::size_t>(num_experts), static_cast<std::size_t>(top_k),
                          static_cast<std::size_t>(in_dim), static_cast<std::size_t>(out_dim),
                          static_cast<std::size_t>(num_shared)};
        spec.validate();
        TileQConfig cfg;
        cfg.grid_rows = static_cast<std::size_t>(grid_rows);
        cfg.grid_cols = static_cast<std::size_t>(grid_cols);
        cfg.rank = static_cast<std::size_t>(rank);
        cfg.bits = bits;
        cfg.group_size = static_cast<std::size_t>(group_size);
        // quantizer 0 rtn, 1 gptq, 2 vq (codebook); gptq / vq run quantize_moe itself
        cfg.quantizer = quantizer == 2 ? ResidualQuantizer::vq
                                       : (quantizer == 1 ? ResidualQuantizer::gptq : ResidualQuantizer::rtn);
        cfg.sub_dim = static_cast<std::size_t>(sub_dim);
        cfg.seed = seed;
        if (quantizer != 0) full_pipeline = 1;
        TileQConfig rc = cfg.resolved(spec);

        SynthResult synth = synth_experts(spec, rc.grid_rows, rc.grid_cols,
                                          static_cast<std::size_t>(planted_rank),
                                          static_cast<float>(mix_scale), static_cast<float>(noise),
                                          seed);
        CounterRng gate_rng(CounterRng::derive(seed, kGateStream));
        DenseMatrix gate = gaussian_matrix(spec.num_experts, spec.in_dim, gate_rng);
        CounterRng calib_rng(CounterRng::derive(seed, kCalibStream));
        DenseMatrix calib;
        if (calib_kind == 0) {
            calib = DenseMatrix(static_cast<std::size_t>(calib_tokens), spec.in_dim);
            for (float& v : calib.data) v = calib_rng.next_unit() < 0.5 ? -1.0f : 1.0f;
        } else if (calib_kind == 1) {
            calib = gaussian_matrix(static_cast<std::size_t>(calib_tokens), spec.in_dim, calib_rng);
        }

        TileQLayer layer;
        if (full_pipeline) {
            layer = quantize_moe(synth.experts, gate, calib, cfg).layer;
        } else {
            // quantize_moe's stage sequence (pipeline.cpp:162-209), minus
            // proxy_loss and the report statistics.
            DenseMatrix stats = calibration_mean_abs(calib, gate, spec);
            ScalingVectors scaling = compute_scaling(stats, rc.scale_exponent);
            FeatureEmbeddings features =
                extract_features(synth.experts, scaling, rc.feature_rank,
                                 CounterRng::derive(rc.seed, kFeatureStream));
            auto ideal = bicluster(features.u_embeddings, features.v_embeddings, rc.grid_rows,
                                   rc.grid_cols, CounterRng::derive(rc.seed, kClusterStream));
            TileAssignment asg = place(ideal, rc.grid_rows, rc.grid_cols);
            DenseMatrix mosaic = build_mosaic(synth.experts, scaling, asg);
            TiledLowRank tiled = decompose_shared(mosaic, rc.rank, rc.power_iters,
                                                  CounterRng::derive(rc.seed, kDecomposeStream),
                                                  asg, scaling);
            mosaic = DenseMatrix{};
            ResidualSet residuals = compute_residuals(synth.experts, tiled);
            layer.spec = spec;
            for (std::size_t k = 0; k < spec.num_experts; ++k)
                layer.quantized.push_back(quantize_rtn(residuals.residuals[k], rc.bits, rc.group_size));
            for (std::size_t s = 0; s < spec.num_shared; ++s)
                layer.shared_quantized.push_back(
                    quantize_rtn(synth.experts.shared[s], rc.bits, rc.group_size));
            layer.tiled = std::move(tiled);
            layer.gate_weights = gate;
        }
        write_artifact(dir, layer);
    });
}

// The comparison layouts of the paper's bench (infer.cpp:187-426) on a GIVEN
// routing: layout 0 fused_2d = lotile_forward, 1 shared_1d =
// baseline_1d_forward on shared_1d_from_tiled_representative, 2 element_wise =
// baseline_elementwise_forward on elementwise_factors_from_tiled, 3
// dequant_only = dequantize every routed expert, as bench() does (y untouched).  The
// factors are prepared outside the measured call, as bench() does
// (infer.cpp:381-387); *dispatches receives dispatch_count() of the call.
int tq_ref_layout(void* hv, int layout, const float* x, std::int64_t batch, const std::int64_t* ids,
                  const float* gates, float* y, std::int64_t* dispatches, char* errbuf, int errlen) {
    auto* h = static_cast<RefHandle*>(hv);
    return guarded(errbuf, errlen, [&] {
        const TileQLayer& layer = h->art.layer;
        const std::size_t k = layer.spec.top_k;
        const std::int64_t in_dim = static_cast<std::int64_t>(layer.spec.in_dim);
        DenseMatrix xm = wrap(x, batch, in_dim);
        RoutingDecision routing;
        routing.batch = static_cast<std::size_t>(batch);
        routing.top_k = k;
        routing.expert_ids.resize(static_cast<std::size_t>(batch) * k);
        routing.gates = DenseMatrix(static_cast<std::size_t>(batch), k);
        for (std::size_t f = 0; f < routing.expert_ids.size(); ++f) {
            routing.expert_ids[f] = static_cast<std::size_t>(ids[f]);
            routing.gates.data[f] = gates[f];
        }
        std::vector<LowRankFactor> ew;
        Shared1DFactors sd;
        if (layout == 1) sd = shared_1d_from_tiled_representative(layer.tiled);
        if (layout == 2) ew = elementwise_factors_from_tiled(layer.tiled);
        reset_dispatch_count();
        DenseMatrix out;
        if (layout == 0) out = lotile_forward(xm, layer.tiled, routing);
        else if (layout == 1) out = baseline_1d_forward(xm, sd, routing);
        else if (layout == 2) out = baseline_elementwise_forward(xm, ew, routing);
        else if (layout == 3) {
            for (const QuantizedExpert& q : layer.quantized) (void)dequantize(q);
        } else {
            throw ParamError("unknown layout " + std::to_string(layout));
        }
        if (dispatches) *dispatches = static_cast<std::int64_t>(dispatch_count());
        if (layout != 3) copy_out(out, y);
    });
}

// The reference's own bench() (infer.cpp:371-426) for one layout: per batch,
// median / p10 / p90 wall ns and the dispatch count (out: 4 doubles per batch).
int tq_ref_bench(void* hv, int layout, const std::int64_t* batches, std::int64_t nb, std::int64_t repeats,
                 std::int64_t warmup, std::uint64_t seed, double* out, char* errbuf, int errlen) {
    auto* h = static_cast<RefHandle*>(hv);
    return guarded(errbuf, errlen, [&] {
        std::vector<std::size_t> bs;
        for (std::int64_t t = 0; t < nb; ++t) bs.push_back(static_cast<std::size_t>(batches[t]));
        const BenchLayout lay = layout == 0 ? BenchLayout::fused_2d
                              : layout == 1 ? BenchLayout::shared_1d
                              : layout == 2 ? BenchLayout::element_wise
                                            : BenchLayout::dequant_only;
        const auto reps = bench(lay, h->art.layer, bs, static_cast<std::size_t>(repeats),
                                static_cast<std::size_t>(warmup), 1, seed);
        for (std::size_t t = 0; t < reps.size(); ++t) {
            out[4 * t + 0] = reps[t].median_ns();
            out[4 * t + 1] = reps[t].p10_ns();
            out[4 * t + 2] = reps[t].p90_ns();
            out[4 * t + 3] = static_cast<double>(reps[t].dispatches);
        }
    });
}

// ---- artifact producer hot spots --------------------------
// estimate_hessian (quant.cpp:116-150), quantize_rtn / quantize_gptq
// (quant.cpp:152-221) and proxy_loss (quant.cpp:325-343) on raw arrays.
// Quantized experts cross as unpacked codes (uint32, rows x cols), per-group
// scales (f32) and zero points (int32), rows x ceil(cols / group_size).

int tq_ref_estimate_hessian(const float* calib, std::int64_t tokens, std::int64_t dim, double damping_fraction,
                            float* h_out, double* damping_out, char* errbuf, int errlen) {
    return guarded(errbuf, errlen, [&] {
        const HessianProxy h = estimate_hessian(wrap(calib, tokens, dim), damping_fraction);
        copy_out(h.h, h_out);
        *damping_out = h.damping;
    });
}

namespace {
void export_quantized(const QuantizedExpert& q, std::uint32_t* codes, float* scales, std::int32_t* zeros) {
    const std::vector<std::uint32_t> c = unpack_codes(q.packed, q.bits, q.code_count());
    std::memcpy(codes, c.data(), c.size() * sizeof(std::uint32_t));
    for (std::size_t t = 0; t < q.grids.size(); ++t) {
        scales[t] = q.grids[t].scale;
        zeros[t] = q.grids[t].zero_point;
    }
}

QuantizedExpert import_quantized(std::int64_t rows, std::int64_t cols, const std::uint32_t* codes,
                                 const float* scales, const std::int32_t* zeros, int bits, std::int64_t gs) {
    QuantizedExpert q;
    q.out_dim = static_cast<std::size_t>(rows);
    q.in_dim = static_cast<std::size_t>(cols);
    q.bits = bits;
    q.mode = QuantMode::scalar;
    q.group_size = static_cast<std::size_t>(gs);
    q.packed = pack_codes(std::vector<std::uint32_t>(codes, codes + rows * cols), bits);
    const std::size_t n = q.out_dim * q.groups_per_row();
    q.grids.resize(n);
    for (std::size_t t = 0; t < n; ++t) q.grids[t] = QuantGrid{scales[t], zeros[t]};
    return q;
}
} // namespace

// method 0: quantize_rtn(r, bits, gs); 1: quantize_gptq(r, {h}, bits, gs)
int tq_ref_quantize(int method, const float* r, std::int64_t rows, std::int64_t cols, const float* h, int bits,
                    std::int64_t gs, std::uint32_t* codes, float* scales, std::int32_t* zeros, char* errbuf,
                    int errlen) {
    return guarded(errbuf, errlen, [&] {
        const DenseMatrix rm = wrap(r, rows, cols);
        QuantizedExpert q;
        if (method == 0) {
            q = quantize_rtn(rm, bits, static_cast<std::size_t>(gs));
        } else {
            HessianProxy hp;
            hp.h = wrap(h, cols, cols);
            q = quantize_gptq(rm, hp, bits, static_cast<std::size_t>(gs));
        }
        export_quantized(q, codes, scales, zeros);
    });
}

int tq_ref_proxy_loss(const float* original, std::int64_t rows, std::int64_t cols, const std::uint32_t* codes,
                      const float* scales, const std::int32_t* zeros, int bits, std::int64_t gs, const float* h,
                      double* out, char* errbuf, int errlen) {
    return guarded(errbuf, errlen, [&] {
        HessianProxy hp;
        hp.h = wrap(h, cols, cols);
        *out = proxy_loss(wrap(original, rows, cols), import_quantized(rows, cols, codes, scales, zeros, bits, gs),
                          hp);
    });
}

int tq_ref_sketch_lowrank(const float* w, std::int64_t rows, std::int64_t cols, std::int64_t rank, int power_iters,
                          std::uint64_t seed, float* left, float* right, float* singulars, char* errbuf, int errlen) {
    return guarded(errbuf, errlen, [&] {
        const LowRankFactor f = sketch_lowrank(wrap(w, rows, cols), static_cast<std::size_t>(rank), power_iters, seed);
        copy_out(f.left, left);
        copy_out(f.right, right);
        std::memcpy(singulars, f.singulars.data(), f.singulars.size() * sizeof(float));
    });
}

} // extern "C"
