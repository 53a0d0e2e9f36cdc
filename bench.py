#!/usr/bin/env python
"""TileQ MoE-layer benchmark (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl tileq|reference]
                    [--workload decode|prefill] [--config c2]

Workload (default, N=1): BASELINE configs[1] -- the Mixtral-8x7B expert layer
(8 experts top-2, h4096, ffn14336, 3-bit TileQ, rank-32 2D-tiled factors,
synthetic weights of that shape) at decode batch 1..64.  One STEP = one full
layer forward (route -> permute -> fused dequant+low-rank tcgen05 expert GEMM
-> gate-weighted combine) at each of B = 1, 2, 4, 8, 16, 32, 64, i.e. 127
tokens; value = 127 * K / (sum of device times).  L2 (126 MB) is flushed
before every forward by writing a 512 MB buffer outside the timed events.
``--workload prefill`` times BASELINE configs[2] (4096 tokens per step).

N>1 (torchrun, one rank per GPU, NCCL): expert parallel (ep.EPLayer) -- each
rank holds K/N experts and its own token batch (weak scaling: every rank runs
the same per-rank sweep), tokens travel by NCCL all-to-all; per-step time is
the max over ranks of the device time.

``--impl reference`` times the reference's own CPU implementation
(oracle/_ref: route + tileq_forward, token-sharded over the host cores) on a
bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

DECODE_BATCHES = (1, 2, 4, 8, 16, 32, 64)
PREFILL_BATCH = 4096
FLUSH_BYTES = 512 << 20


def _env_int(name, default):
    v = os.environ.get(name)
    return int(v) if v not in (None, "") else default


# ---------------------------------------------------------------------------
# clocks (nvidia-smi sampled during the timed region)
# ---------------------------------------------------------------------------

class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm, mx, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[3:7]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# algorithmic bytes / flops, stated in DESIGN.md
# ---------------------------------------------------------------------------

class Geometry:
    def __init__(self, info):
        self.K, self.k, self.i, self.o = (info[n] for n in ("num_experts", "top_k", "in_dim", "out_dim"))
        self.S, self.r, self.bits, self.g = (info[n] for n in ("num_shared", "rank", "bits", "group_size"))
        self.M, self.N = info["grid_rows"], info["grid_cols"]
        self.G = -(-self.i // self.g)

    def residual_bytes(self):
        """codes + f16 scales + packed zeros of one o x i matrix."""
        return self.o * self.i * self.bits // 8 + 2 * self.o * self.G + -(-self.o * self.G * self.bits // 8)

    def gemm_bytes(self, ids: np.ndarray, placement_rows: np.ndarray) -> int:
        """Algorithmic HBM bytes of one fused expert-GEMM launch: residual
        payload of each distinct active expert (+ shared), the int8 u-block of
        each distinct tile row p touched, the fp16 activation rows read and the
        f32 expert-output rows written."""
        act = np.unique(ids)
        ps = np.unique(placement_rows[act])
        B = ids.shape[0]
        n_rows = B * self.k
        return int((len(act) + self.S) * self.residual_bytes() + len(ps) * self.o * self.r
                   + 2 * (n_rows + B * self.S) * self.i + 4 * (n_rows + B * self.S) * self.o)

    def layer_bytes(self, ids: np.ndarray, placement: np.ndarray, general: bool) -> int:
        """SURVEY §8(d) whole-forward algorithmic bytes."""
        act = np.unique(ids)
        ps = np.unique(placement[act, 0])
        qs = np.unique(placement[act, 1])
        B = ids.shape[0]
        b = (len(act) + self.S) * self.residual_bytes() + len(ps) * self.o * self.r + len(qs) * self.r * self.i
        if general:
            b += 4 * self.i * len(act)
        return int(b + 4 * self.K * self.i + 4 * B * self.i + 4 * B * self.o)

    def flops(self, B: int) -> float:
        return 2.0 * B * self.k * (self.o * self.i + self.r * self.i + self.r * self.o) + 2.0 * B * self.S * self.o * self.i


def placement_of(artifact_dir: str) -> np.ndarray:
    with open(os.path.join(artifact_dir, "manifest.json")) as f:
        man = json.load(f)
    ent = man["tensors"]["placement"]
    with open(os.path.join(artifact_dir, ent["file"]), "rb") as f:
        return np.frombuffer(f.read(), np.uint16).reshape(-1, 2).astype(np.int64)


def measured_peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            m = json.load(f)
        return float(m["hbm_gbs"]), float(m["bf16_tflops"]), float(m.get("bf16_tflops_sustained", m["bf16_tflops"])), "measured"
    except (OSError, KeyError, ValueError):
        return 6650.0, 1590.0, 1400.0, "fallback"


def traffic_from_profiles(workload: str, batches):
    """dram__bytes_read+write per launch of the fused GEMM from the committed
    ncu --set full captures (profiles/gemm_traffic.json): the mean over the
    workload's batch sizes when every one was captured, else the captured
    sizes by batch (with the source), else None."""
    try:
        with open(os.path.join(REPO, "profiles", "gemm_traffic.json")) as f:
            ent = json.load(f).get(workload)
    except (OSError, ValueError):
        return None
    if not ent:
        return None
    per = ent.get("per_batch_bytes", {})
    if all(str(b) in per for b in batches):
        return float(np.mean([per[str(b)] for b in batches]))
    return {"per_batch_bytes": per, "source": ent.get("source")}


# ---------------------------------------------------------------------------
# workload
# ---------------------------------------------------------------------------

def make_tokens(B: int, i: int, seed: int) -> np.ndarray:
    return np.random.default_rng(seed).standard_normal((B, i), dtype=np.float32)


def artifact_for(config: str, rank: int, world: int) -> str:
    from paper_2605_09281_b200 import synth
    root = os.environ.get("TILEQ_ARTIFACT_ROOT", "/tmp/tileq_artifacts")
    path = synth.config_path(config, root)
    if rank == 0:
        synth.ensure_config(config, root=root)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    return path


def cpu_info() -> dict:
    """nproc (cores usable by this process) and the CPU model (BASELINE.md asks for both)."""
    nproc = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"nproc": nproc, "cpu_model": model}


def host_threads(B: int, per_thread_bytes: int) -> int:
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    try:
        import psutil
        avail = psutil.virtual_memory().available
    except Exception:
        avail = 16 << 30
    by_mem = max(1, int(0.6 * avail // max(per_thread_bytes, 1)))
    return max(1, min(cores, B, by_mem))


def run_reference_sample(artifact_dir: str, B: int, i: int, o: int, K: int, S: int, seed: int = 7):
    """One bounded sample: route + tileq_forward (oracle/_ref) on B tokens,
    token-sharded over the host cores (each shard dequantizes all K+S experts:
    ~4*o*i*(K+S) bytes of working memory per thread, which caps the threads)."""
    from oracle.oracle import RefLib
    ref = RefLib()
    R = ref.load(artifact_dir)
    x = make_tokens(B, i, seed)
    T = host_threads(B, 4 * o * i * (K + S) + (64 << 20))
    t0 = time.perf_counter()
    R.forward(x, mode=0, threads=T)
    dt = time.perf_counter() - t0
    return dt, T, R, x


# ---------------------------------------------------------------------------
# reference arm
# ---------------------------------------------------------------------------

def bench_reference(args, rank, world):
    """The reference's own CPU path (oracle/_ref = the unmodified reference C++:
    route + tileq_forward) on the box's host cores.  A decode step of the GPU
    arm is the B = 1..64 sweep (127 tokens); one reference call costs ~10 s
    whatever B is (every call dequantizes all experts, infer.cpp:45-49), so a
    reference step is ONE 64-token batch -- the CPU's most favourable point of
    the sweep, labelled as such.  Every step of --steps is timed (the time
    budget only stops a run that would not finish, and then `steps` says so)."""
    if rank != 0:
        return 0
    from oracle.oracle import RefLib, ref_available
    if not ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libtileq_ref.so missing (built from /root/reference by __graft_entry__.build())"}))
        return 0
    from paper_2605_09281_b200 import synth
    K, top_k, i, o, S, bits, r, g = synth.CONFIGS[args.config]
    art = artifact_for(args.config, 0, 1)
    B = 64 if args.workload == "decode" else 256
    ref = RefLib()
    R = ref.load(art)
    T = host_threads(B, 4 * o * i * (K + S) + (64 << 20))
    budget = float(os.environ.get("TILEQ_REF_BUDGET_S", "420"))
    t_start = time.perf_counter()
    n_warm = min(args.warmup, 1)
    for w in range(n_warm):
        R.forward(make_tokens(B, i, 1000 + w), mode=0, threads=T)
    times = []
    for s_ in range(args.steps):
        x = make_tokens(B, i, 2000 + s_)
        t0 = time.perf_counter()
        R.forward(x, mode=0, threads=T)
        times.append(time.perf_counter() - t0)
        if time.perf_counter() - t_start > budget:
            break
    sec = float(np.median(times))
    val = B / sec
    info = cpu_info()
    sample = (f"route + tileq_forward (reference C++, oracle/_ref) on ONE {B}-token batch of {args.config} per step "
              f"(the {'B=64 point of the decode sweep' if args.workload == 'decode' else '256-token sample of the prefill batch'}), "
              f"token-sharded over {T} threads; {len(times)} timed steps (median), {n_warm} warm-up")
    cfg = workload_config(args, world)
    cfg["reference_step"] = f"one {B}-token batch per step (tokens_per_step {B})"
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": "tokens/s", "n_gpus": world,
            "steps": len(times), "steps_requested": args.steps, "warmup": n_warm, "ms_per_step": sec * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64/f32 (CPU)",
            "data": "synthetic", "config": cfg,
            "cpu_baseline": {"value": val, "unit": "tokens/s", "cores": T, "kind": "reference", "sample": sample, **info},
            "e2e": {"value": val, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


METRIC = "TileQ MoE-layer tokens/s (decode+prefill), % of HBM/tensor roofline"


def workload_config(args, world):
    if args.workload == "decode":
        wl = f"{args.config} Mixtral-8x7B expert layer (8 experts top-2, h4096, ffn14336), 3-bit TileQ r=32, decode sweep B=1,2,4,8,16,32,64 per step"
        batches = list(DECODE_BATCHES)
    else:
        wl = f"{args.config} Mixtral-8x7B expert layer prefill, {PREFILL_BATCH} tokens per rank per step"
        batches = [PREFILL_BATCH]
    return {"workload": wl, "batches_per_rank": batches, "tokens_per_step": world * sum(batches),
            "parallelism": f"ep{world}" if world > 1 else "single-gpu",
            "l2": "flushed (512 MB write) before every forward, outside the timed events",
            "weights": "synthetic artifact of the named shape (reference wire format), folded tier"}


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def bench_tileq(args, rank, world, local_rank):
    import torch
    import paper_2605_09281_b200 as tq
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    art = artifact_for(args.config, rank, world)
    if world > 1:
        import torch.distributed as dist
        from paper_2605_09281_b200.ep import EPLayer
        ep = EPLayer(art, device=local_rank)
        if args.workload == "decode":
            # fixed-capacity exchange (equal splits, device-side counts): no host round trip
            ep.slab = max(DECODE_BATCHES) * ep.top_k
        L = ep.stages
        fwd = lambda x, out: ep.forward(x, out=out)  # noqa: E731
    else:
        ep = None
        L = tq.Layer(art, device=local_rank)
        fwd = lambda x, out: L.forward(x, out=out)  # noqa: E731
    info = L.info
    geo = Geometry(info)
    placement = placement_of(art)
    batches = list(DECODE_BATCHES) if args.workload == "decode" else [PREFILL_BATCH]
    L.reserve(max(batches) * (world if world > 1 else 1))
    xs = [torch.from_numpy(make_tokens(B, geo.i, 100 * rank + B)).to(dev) for B in batches]
    ys = [torch.empty((B, geo.o), dtype=torch.float32, device=dev) for B in batches]
    flush = torch.empty(FLUSH_BYTES, dtype=torch.uint8, device=dev)

    def barrier():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    # routing of the run (deterministic in x): algorithmic bytes per forward
    gemm_bytes, layer_bytes = [], []
    for x in xs:
        ids, _ = L.route(x)
        idn = ids.cpu().numpy()
        gemm_bytes.append(geo.gemm_bytes(idn, placement[:, 0]) if world == 1 else 0)
        layer_bytes.append(geo.layer_bytes(idn, placement, info["tier_general"] > 0))

    def one_step(timed: bool):
        evs = []
        for x, y in zip(xs, ys):
            flush.zero_()
            if timed:
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                fwd(x, y)
                b.record()
                evs.append((a, b))
            else:
                fwd(x, y)
        return evs

    clocks = ClockSampler(local_rank).start() if rank == 0 else None
    for _ in range(args.warmup):
        one_step(False)
    # keep the GPU busy (untimed) until nvidia-smi has produced samples, so the
    # clock record covers a loaded GPU; the sampler keeps running through the
    # timed region
    settle = 0
    t_settle = time.time()
    while True:
        ready = clocks is None or len(clocks.lines) >= 3 or time.time() - t_settle > 5.0
        if world > 1:
            import torch.distributed as dist
            flag = torch.tensor([1 if ready else 0], device=dev)
            dist.all_reduce(flag, op=dist.ReduceOp.MIN)
            ready = bool(flag.item())
        if ready:
            break
        one_step(False)
        torch.cuda.synchronize()
        settle += 1
    barrier()
    L.reset_launch_count()
    barrier()
    all_evs = [one_step(True) for _ in range(args.steps)]   # the measurement (CUDA-graph replays)
    barrier()
    launches = L.launch_count()
    clk = clocks.stop() if clocks else None
    # second pass over the same steps with the GEMM bracketed by events (graphs
    # off for this pass only): the dominant kernel's device time for the roofline
    L.gemm_timing(True)
    for _ in range(args.steps):
        one_step(False)
    torch.cuda.synchronize()
    gemm_ms, gemm_n = L.gemm_time()
    L.gemm_timing(False)
    gemm_passes = args.steps
    per_b_ms = np.zeros(len(batches))
    for evs in all_evs:
        for j, (a, b) in enumerate(evs):
            per_b_ms[j] += a.elapsed_time(b)
    total_ms = float(per_b_ms.sum())
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    tokens_per_step = world * sum(batches)
    value = tokens_per_step / (ms_per_step * 1e-3)

    # ---- e2e: host buffers through the public API, copies inside the timed region
    e2e = e2e_measure(args, L, ep, xs, batches, geo, dev, flush, world)

    if rank != 0:
        return 0
    hbm, tf_burst, tf_sust, peak_kind = measured_peaks()
    # dominant kernel = the fused expert GEMM (one launch per forward)
    launches_per_fwd = gemm_n / max(1, gemm_passes * len(batches))
    gemm_avg_ms = gemm_ms / max(gemm_n, 1)
    if args.workload == "decode":
        algo = float(np.mean(gemm_bytes)) if world == 1 else None
        achieved = (algo / (gemm_avg_ms * 1e-3) / 1e9) if algo else None
        roof = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                "frac": (achieved / hbm) if achieved else None, "traffic": traffic_from_profiles("decode", batches),
                "kernel": "dec_gemm_kernel<3,32|64> (fused dequant + low-rank tcgen05 expert GEMM, decode path)",
                "algorithmic_bytes_per_launch": algo, "avg_launch_ms": gemm_avg_ms,
                "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind}, burst copy)",
                "share_of_step": (gemm_ms / gemm_passes) / ms_per_step if ms_per_step else None}
    else:
        fl = geo.flops(PREFILL_BATCH)
        achieved = fl / (gemm_avg_ms * 1e-3) / 1e12
        roof = {"bound": "tensor", "achieved": achieved, "peak": tf_burst, "unit": "TFLOP/s",
                "frac": achieved / tf_burst, "traffic": traffic_from_profiles("prefill", batches),
                "kernel": "tq_gemm (fused dequant + low-rank tcgen05 expert GEMM)",
                "algorithmic_flops_per_launch": fl, "avg_launch_ms": gemm_avg_ms,
                "peak_source": f"MEASURED_PEAKS.json bf16_tflops ({peak_kind}, burst cuBLAS)",
                "share_of_step": (gemm_ms / gemm_passes) / ms_per_step if ms_per_step else None}
    per_b = {str(B): {"us": per_b_ms[j] / args.steps * 1e3,
                      "tokens_per_s": B / (per_b_ms[j] / args.steps * 1e-3),
                      "layer_bytes": layer_bytes[j],
                      "layer_hbm_frac": layer_bytes[j] / (per_b_ms[j] / args.steps * 1e-3) / 1e9 / hbm}
             for j, B in enumerate(batches)}
    line = {"metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f16 x f16 -> f32 (3-bit codes dequantized in registers)",
            "data": "synthetic", "config": workload_config(args, world), "roofline": roof,
            "per_batch": per_b, "e2e": e2e, "gpu_launches": int(launches),
            "gpu_launches_per_forward": launches / max(1, args.steps * len(batches)),
            "gemm_launches_per_forward": launches_per_fwd, "clocks": clk, "clock_settle_steps": settle}
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_leg(args, art, geo)
    if world == 1 and args.workload == "decode" and not args.no_prefill:
        line["prefill"] = prefill_leg(args, L, geo, dev, flush, art)
    print(json.dumps(line), flush=True)
    return 0


def prefill_leg(args, L, geo, dev, flush, art):
    """BASELINE configs[2] on the same layer: one 4096-token forward per step
    (c3 is c2's shape), device time by CUDA events with L2 flushed before every
    forward; roofline of the dominant kernel (the grouped tcgen05 expert GEMM)
    against the measured bf16 burst peak; e2e through tq_forward_host; a
    bounded reference CPU sample (256 tokens)."""
    import torch
    B = PREFILL_BATCH
    L.reserve(B)
    x = torch.from_numpy(make_tokens(B, geo.i, 4242)).to(dev)
    y = torch.empty((B, geo.o), dtype=torch.float32, device=dev)
    steps = max(3, min(args.steps, 10))
    for _ in range(3):
        flush.zero_()
        L.forward(x, out=y)
    torch.cuda.synchronize()
    L.reset_launch_count()
    tot = 0.0
    for _ in range(steps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        L.forward(x, out=y)
        b.record()
        b.synchronize()
        tot += a.elapsed_time(b)
    launches = L.launch_count()
    ms = tot / steps
    L.gemm_timing(True)
    for _ in range(steps):
        flush.zero_()
        L.forward(x, out=y)
    torch.cuda.synchronize()
    gemm_ms, gemm_n = L.gemm_time()
    L.gemm_timing(False)
    gemm_avg = gemm_ms / max(gemm_n, 1)
    hbm, tf_burst, tf_sust, peak_kind = measured_peaks()
    fl = geo.flops(B)
    achieved = fl / (gemm_avg * 1e-3) / 1e12
    # e2e: host buffers, H2D of x and D2H of y inside the timed region
    hx = torch.from_numpy(make_tokens(B, geo.i, 4242)).pin_memory()
    hy = torch.empty((B, geo.o), dtype=torch.float32).pin_memory()
    L.forward_host(hx.numpy(), out=hy.numpy())
    e_tot = 0.0
    for _ in range(3):
        flush.zero_()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        L.forward_host(hx.numpy(), out=hy.numpy())
        b.record()
        b.synchronize()
        e_tot += a.elapsed_time(b)
    e_ms = e_tot / 3
    out = {"workload": f"configs[2]: {args.config} shape prefill, {B} tokens per step", "value": B / (ms * 1e-3),
           "unit": "tokens/s", "steps": steps, "warmup": 3, "ms_per_step": ms,
           "roofline": {"bound": "tensor", "achieved": achieved, "peak": tf_burst, "unit": "TFLOP/s",
                        "frac": achieved / tf_burst, "traffic": traffic_from_profiles("prefill", [B]),
                        "kernel": "gemm_kernel<b,64,2,192,1> (grouped fused dequant + low-rank tcgen05 expert GEMM)",
                        "algorithmic_flops_per_launch": fl, "avg_launch_ms": gemm_avg,
                        "peak_source": f"MEASURED_PEAKS.json bf16_tflops ({peak_kind}, burst cuBLAS)",
                        "share_of_step": gemm_avg * (gemm_n / max(steps, 1)) / ms},
           "gpu_launches_per_forward": launches / steps,
           "e2e": {"value": B / (e_ms * 1e-3), "unit": "tokens/s", "ms_per_step": e_ms, "steps": 3,
                   "h2d_bytes_per_step": 4 * B * geo.i, "d2h_bytes_per_step": 4 * B * geo.o,
                   "api": "Layer.forward_host -> tq_forward_host (C-ABI, host f32 in/out)"}}
    if not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_sample(art, 256, geo, args.config + " (prefill sample)")
    return out


def e2e_measure(args, L, ep, xs, batches, geo, dev, flush, world):
    """Same metric through the public API with pinned HOST buffers: the H2D of
    x and the D2H of y are inside the timed region (tq_forward_host at N=1)."""
    import torch
    hx = [torch.empty(x.shape, dtype=torch.float32, pin_memory=True) for x in xs]
    hy = [torch.empty((x.shape[0], geo.o), dtype=torch.float32, pin_memory=True) for x in xs]
    for h, x in zip(hx, xs):
        h.copy_(x.cpu())
    steps = max(1, min(args.steps, 10))

    def call(j):
        if ep is None:
            L.forward_host(hx[j].numpy(), out=hy[j].numpy())
        else:
            xd = hx[j].to(dev, non_blocking=True)
            y = ep.forward(xd)
            hy[j].copy_(y, non_blocking=True)
            torch.cuda.current_stream().synchronize()

    for j in range(len(xs)):
        call(j)
    torch.cuda.synchronize()
    tot = 0.0
    for _ in range(steps):
        for j in range(len(xs)):
            flush.zero_()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            call(j)
            b.record()
            b.synchronize()
            tot += a.elapsed_time(b)
    if world > 1:
        t = torch.tensor([tot], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        tot = float(t.item())
    ms = tot / steps
    toks = world * sum(batches)
    return {"value": toks / (ms * 1e-3), "unit": "tokens/s", "ms_per_step": ms, "steps": steps,
            "h2d_bytes_per_step": int(sum(4 * x.numel() for x in xs)),
            "d2h_bytes_per_step": int(sum(4 * x.shape[0] * geo.o for x in xs)),
            "api": "Layer.forward_host -> tq_forward_host (C-ABI, host f32 in/out)" if ep is None
            else "pinned H2D + EPLayer.forward + D2H"}


def cpu_baseline_leg(args, art, geo):
    from oracle.oracle import ref_available
    if not ref_available():
        return {"value": None, "unit": "tokens/s", "cores": 0, "kind": "reference",
                "sample": "unavailable: oracle/_ref not built"}
    B = 64 if args.workload == "decode" else 256
    return cpu_sample(art, B, geo, args.config)


def cpu_sample(art, B, geo, name):
    dt, T, _, _ = run_reference_sample(art, B, geo.i, geo.o, geo.K, geo.S)
    return {"value": B / dt, "unit": "tokens/s", "cores": T, "kind": "reference",
            "sample": f"one route + tileq_forward call of the reference C++ (oracle/_ref) on {B} tokens of "
                      f"{name}, token-sharded over {T} host threads ({dt:.1f} s)", **cpu_info()}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="tileq", choices=["tileq", "reference"])
    ap.add_argument("--workload", default="decode", choices=["decode", "prefill"])
    ap.add_argument("--config", default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-prefill", action="store_true", help="decode workload only (skip the prefill object)")
    args = ap.parse_args()
    if args.config is None:
        args.config = "c2" if args.workload == "decode" else "c3"
    args.warmup = max(args.warmup, 3) if args.impl == "tileq" else args.warmup
    world = _env_int("WORLD_SIZE", 1)
    rank = _env_int("RANK", 0)
    local_rank = _env_int("LOCAL_RANK", 0)
    if world > 1:
        import torch
        import torch.distributed as dist
        if args.impl == "reference":
            if rank != 0:
                return 0
            world_ref = world
            return bench_reference(args, 0, world_ref)
        # one rank per GPU over NCCL; TILEQ_DIST_BACKEND=gloo runs the same EP path
        # with host-staged exchanges (lets several ranks share one GPU for testing)
        backend = os.environ.get("TILEQ_DIST_BACKEND", "nccl")
        dev_idx = local_rank % max(1, torch.cuda.device_count())
        torch.cuda.set_device(dev_idx)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev_idx))
        else:
            dist.init_process_group(backend)
        try:
            return bench_tileq(args, rank, world, dev_idx)
        finally:
            dist.destroy_process_group()
    if args.impl == "reference":
        return bench_reference(args, 0, 1)
    # a device fault fails the run (non-zero exit): a faulting kernel posts no number
    return bench_tileq(args, 0, 1, local_rank)

if __name__ == "__main__":
    sys.exit(main())
