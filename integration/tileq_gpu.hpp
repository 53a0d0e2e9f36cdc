// tileq_gpu.hpp -- the reference-side C++ shim over libtileq_b200.so.
//
// A maintainer of the reference library adds this header and tileq_gpu.cpp to
// their build (include path: the reference's include/, plus this repo's
// include/ for tileq_b200.h; link: libtileq_b200.so).  Every function keeps
// the signature of the reference function it stands for, on the reference's
// own types, so a caller switches engines by namespace alone:
//
//   tileq::gpu::route            <- tileq::route            include/tileq/moe.hpp:53
//   tileq::gpu::qmoe_forward     <- tileq::qmoe_forward     include/tileq/infer.hpp:52-53
//   tileq::gpu::lotile_forward   <- tileq::lotile_forward   include/tileq/infer.hpp:68-69
//   tileq::gpu::tileq_forward    <- tileq::tileq_forward    include/tileq/infer.hpp:72-73
//   tileq::gpu::forward_from_artifact <- _tileq.forward_from_artifact  bindings/py_module.cpp:112-117
//   tileq::gpu::reset_dispatch_count / dispatch_count <- infer.hpp:37-38 (GPU analogue:
//                                    kernel launches, constant in the batch size)
//   tileq::gpu::estimate_hessian <- tileq::estimate_hessian include/tileq/quant.hpp:67
//   tileq::gpu::quantize_rtn     <- tileq::quantize_rtn     include/tileq/quant.hpp:74
//   tileq::gpu::quantize_gptq    <- tileq::quantize_gptq    include/tileq/quant.hpp:85-86
//   tileq::gpu::proxy_loss       <- tileq::proxy_loss       include/tileq/quant.hpp:104
//   tileq::gpu::sketch_lowrank   <- tileq::sketch_lowrank   include/tileq/lowrank.hpp:21-30
//                                    (the artifact producer's hot spots; bit-identical results)
//
// Failures surface as the reference's exception types (errors.hpp:13-50):
// the C-ABI status is mapped back to ShapeError / ParamError / FormatError /
// IoError / ... with the engine's message, so CHECK_THROWS_AS-style tests
// keep working.  Device-resident layers are cached per TileQLayer (address +
// content fingerprint) or artifact directory, so repeated forwards of one
// layer upload it once.
#pragma once

#include <cstdint>
#include <string>

#include "tileq/infer.hpp"
#include "tileq/lowrank.hpp"
#include "tileq/moe.hpp"
#include "tileq/quant.hpp"

namespace tileq::gpu {

RoutingDecision route(const DenseMatrix& x, const DenseMatrix& gate_weights, std::size_t top_k);

DenseMatrix qmoe_forward(const DenseMatrix& x, const TileQLayer& layer, const RoutingDecision& routing);

/// Low-rank half only, from the tiled factors alone (like the reference): the
/// shim serves it from a layer whose residuals are all-zero codes.
DenseMatrix lotile_forward(const DenseMatrix& x, const TiledLowRank& tiled, const RoutingDecision& routing,
                           int threads = 1);

DenseMatrix tileq_forward(const DenseMatrix& x, const TileQLayer& layer, const RoutingDecision& routing);

/// route + tileq_forward on an artifact directory (read and validated by the
/// engine's own loader, io.cpp:679-813 semantics).
DenseMatrix forward_from_artifact(const std::string& dir, const DenseMatrix& x);

void reset_dispatch_count();
std::uint64_t dispatch_count();

/// CUDA device the shim places layers on (default 0).
void set_device(int device);
/// Free every cached device-resident layer.
void clear_cache();

// artifact producer: same results as the reference, bit for bit
HessianProxy estimate_hessian(const DenseMatrix& calib_inputs, double damping_fraction);
QuantizedExpert quantize_rtn(const DenseMatrix& r, int bits, std::size_t group_size);
QuantizedExpert quantize_gptq(const DenseMatrix& r, const HessianProxy& h, int bits, std::size_t group_size);
double proxy_loss(const DenseMatrix& original, const QuantizedExpert& q, const HessianProxy& h);
LowRankFactor sketch_lowrank(const DenseMatrix& w, std::size_t rank, int power_iters, std::uint64_t seed);

}  // namespace tileq::gpu
