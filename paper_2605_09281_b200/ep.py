"""Expert-parallel TileQ layer: one process per GPU, NCCL all-to-all over NVLink.

SURVEY.md §8(e).  Routed experts are split into contiguous, balanced blocks
(rank r owns [r*K//W, (r+1)*K//W)); the router, factor blocks and shared
experts are replicated.  Each rank routes its own tokens, then

  1. permute    -- stable counting sort by expert id (bit-exact, §8a15); as
                   expert blocks are contiguous per rank, the permuted slots
                   are already grouped by destination rank
  2. rows       -- fp16 token rows + fp16 extension rows (group sums and the
                   rank-r projection X·A computed at home, the factors being
                   replicated) written straight into the send layout
  3. counts     -- all-to-all of a [W, E_max] int32 count matrix (per
                   destination: rows per owned expert)
  4. dispatch   -- all-to-all of the rows
  5. experts    -- fused dequant + tcgen05 GEMM on received rows, one segment
                   per (source rank, local expert)
  6. return     -- all-to-all of the f32 expert outputs back to the home rank
  7. combine    -- y[b] = sum_{t ascending} g[b,t]·Y[inv[b,t]] + shared,
                   the reference's order (moe.cpp:106-133, moe.hpp:55-58)

The orchestration is written against two small interfaces so the same code
runs (a) on GPUs with torch.distributed/NCCL and the sm_100a stages of
``Layer``, and (b) in the CPU tests with gloo and checker-backed stages.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np


def expert_bounds(num_experts: int, world: int) -> list:
    """Contiguous balanced expert blocks: rank r owns [b[r], b[r+1])."""
    if world < 1 or num_experts < world:
        from . import ParamError
        raise ParamError(f"expert parallel: {num_experts} experts over {world} ranks")
    return [(r * num_experts) // world for r in range(world + 1)]


def owner_of(bounds: list, expert: int) -> int:
    for r in range(len(bounds) - 1):
        if bounds[r] <= expert < bounds[r + 1]:
            return r
    raise ValueError(expert)


def send_plan(offsets: np.ndarray, bounds: list):
    """From permute offsets (K+1, host) to (rows per destination rank,
    [W, E_max] count matrix with row d = counts of d's experts)."""
    W = len(bounds) - 1
    emax = max(bounds[r + 1] - bounds[r] for r in range(W))
    counts = np.zeros((W, emax), np.int32)
    rows = np.zeros(W, np.int64)
    per_expert = np.diff(offsets.astype(np.int64))
    for d in range(W):
        c = per_expert[bounds[d]:bounds[d + 1]]
        counts[d, :len(c)] = c
        rows[d] = c.sum()
    return rows, counts


def recv_segments(recv_counts: np.ndarray, n_local: int):
    """Received rows arrive grouped by source rank, then by local expert.
    Returns (rows per source, int64 [n, 3] segments (local expert, first row, count))."""
    W = recv_counts.shape[0]
    segs = []
    per_src = np.zeros(W, np.int64)
    row = 0
    for s in range(W):
        for j in range(n_local):
            c = int(recv_counts[s, j])
            if c:
                segs.append((j, row, c))
            row += c
            per_src[s] += c
    return per_src, np.asarray(segs, np.int64).reshape(-1, 3)


# ---------------------------------------------------------------------------
# communication backends
# ---------------------------------------------------------------------------

class TorchComm:
    """torch.distributed all-to-all (NCCL on B200s, gloo in the CPU tests)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        # gloo moves host tensors only: stage device tensors through the host
        self.stage = dist.get_backend(group) == "gloo"

    def _a2a(self, out, inp, **kw):
        if self.stage and inp.is_cuda:
            o = out.cpu()
            self.dist.all_to_all_single(o, inp.cpu(), group=self.group, **kw)
            out.copy_(o)
        else:
            self.dist.all_to_all_single(out, inp, group=self.group, **kw)

    def all_to_all_counts(self, counts):
        """counts: torch int32 [W, E_max] (device of the backend) -> same shape."""
        import torch
        out = torch.empty_like(counts)
        self._a2a(out, counts.contiguous())
        return out

    def all_to_all_rows(self, send, send_rows, recv_rows):
        import torch
        recv = torch.empty((int(sum(recv_rows)),) + tuple(send.shape[1:]), dtype=send.dtype, device=send.device)
        self._a2a(recv, send.contiguous(), output_split_sizes=[int(v) for v in recv_rows],
                  input_split_sizes=[int(v) for v in send_rows])
        return recv


# ---------------------------------------------------------------------------
# the layer
# ---------------------------------------------------------------------------

@dataclass
class _Pending:
    x: object
    ids: object
    gates: object
    inv: object
    send_rows: np.ndarray
    recv_rows: np.ndarray


class EPLayer:
    """A TileQ layer sharded by expert over the ranks of ``comm``.

    ``stages`` defaults to the sm_100a engine (a ``Layer`` holding this rank's
    expert block); tests pass checker-backed stages with the same methods:
    route, permute, ep_dispatch_rows, ep_expert_rows, ep_combine.
    """

    def __init__(self, artifact_dir: Optional[str] = None, comm=None, device: Optional[int] = None,
                 stages=None, num_experts: Optional[int] = None, path: str = "full", slab: Optional[int] = None):
        self.comm = comm if comm is not None else TorchComm()
        W, r = self.comm.world, self.comm.rank
        if stages is None:
            import json
            import os
            from . import Layer, FormatError, IoError
            try:
                with open(os.path.join(artifact_dir, "manifest.json")) as f:
                    K = int(json.load(f)["meta"]["spec"]["num_experts"])
            except OSError as e:
                raise IoError(f"cannot read manifest: {e}") from e
            except (KeyError, TypeError, ValueError) as e:
                raise FormatError(f"manifest: {e}") from e
            self.bounds = expert_bounds(K, W)
            stages = Layer(artifact_dir, device=device if device is not None else 0,
                           expert_range=(self.bounds[r], self.bounds[r + 1]))
        else:
            K = num_experts if num_experts is not None else stages.num_experts
            self.bounds = expert_bounds(K, W)
        self.stages = stages
        self.num_experts = K
        self.top_k = stages.top_k
        self.out_dim = stages.out_dim
        self.in_dim = stages.in_dim
        self.path = path
        self.e_begin, self.e_end = self.bounds[r], self.bounds[r + 1]
        # slab: fixed per-destination row capacity (decode sizes).  Every all-to-all then
        # has equal, host-known splits and the receive side builds its work units from
        # the device-resident counts: a forward with no host round trip.  All ranks
        # must agree on it (and on B * top_k <= slab).
        self.slab = slab

    # -- phases (usable one by one by an emulator that steps several ranks) --
    def phase_dispatch(self, x):
        """route + permute + rows.  Returns (pending state, send rows x, send rows ext, count matrix)."""
        import torch
        S = self.stages
        ids, gates = S.route(x)
        perm, offsets, inv = S.permute(ids)
        xrows, erows = S.ep_dispatch_rows(x, ids, perm, self.path)
        send_rows, counts = send_plan(offsets.cpu().numpy(), self.bounds)
        pend = _Pending(x, ids, gates, inv, send_rows, None)
        return pend, xrows, erows, torch.from_numpy(counts)

    def phase_experts(self, recv_counts: np.ndarray, xrecv, erecv):
        per_src, segs = recv_segments(recv_counts, self.e_end - self.e_begin)
        y = self.stages.ep_expert_rows(xrecv, erecv, segs, self.path)
        return y, per_src

    def phase_combine(self, pend: _Pending, yback, out=None):
        return self.stages.ep_combine(pend.x, yback, pend.inv, pend.gates, self.path, out=out)

    # -- fixed-capacity (slab) phases: no host round trip -------------------
    def slab_dispatch(self, x):
        """route + permute + rows into the [W * slab, xw + ew] send buffer.  Returns
        (pending state, send buffer, [W, E_max] int32 count matrix, slot -> slab index)."""
        import torch
        S, W, C, k = self.stages, self.comm.world, self.slab, self.top_k
        B = x.shape[0]
        if B * k > C:
            from . import ShapeError
            raise ShapeError(f"expert parallel slab: {B} tokens x top_k {k} exceed the slab capacity {C}")
        dev = x.device
        ids, gates = S.route(x)
        perm, offsets, inv = S.permute(ids)
        xrows, erows = S.ep_dispatch_rows(x, ids, perm, self.path)
        xw, ew = xrows.shape[1], erows.shape[1]
        off = offsets.to(dev).long()
        starts = off[torch.tensor(self.bounds, device=dev)]           # first permuted slot per destination
        pos = torch.arange(B * k, device=dev)
        dest = torch.searchsorted(starts[1:].contiguous(), pos, right=True)
        idx = dest * C + (pos - starts[dest])
        send = torch.zeros((W * C, xw + ew), dtype=xrows.dtype, device=dev)
        send[idx, :xw] = xrows
        send[idx, xw:] = erows.to(xrows.dtype)
        emax = max(self.bounds[d + 1] - self.bounds[d] for d in range(W))
        ej = torch.tensor([[self.bounds[d] + j if self.bounds[d] + j < self.bounds[d + 1] else -1 for j in range(emax)]
                           for d in range(W)], device=dev)
        per_e = off[1:] - off[:-1]
        counts = torch.where(ej >= 0, per_e[ej.clamp(min=0)], torch.zeros_like(ej)).to(torch.int32)
        pend = _Pending(x, ids, gates, inv, None, None)
        return pend, send, counts, idx, xw

    def forward_slab(self, x, out=None):
        import torch
        c, C, W = self.comm, self.slab, self.comm.world
        pend, send, counts, idx, xw = self.slab_dispatch(x)
        recv_counts = c.all_to_all_counts(counts)
        recv = c.all_to_all_rows(send, [C] * W, [C] * W)
        y = self.stages.ep_expert_rows_slab(recv, W, C, recv_counts, self.path)
        yback = c.all_to_all_rows(y, [C] * W, [C] * W)
        inv_slab = idx[pend.inv.to(idx.device).long()].to(torch.int32)
        return self.stages.ep_combine(pend.x, yback, inv_slab, pend.gates, self.path, out=out)

    # -- the collective forward ----------------------------------------------
    def forward(self, x, out=None):
        """y = tileq_forward(x) for this rank's tokens, experts computed where they live."""
        if self.slab is not None:
            return self.forward_slab(x, out=out)
        c = self.comm
        pend, xrows, erows, counts = self.phase_dispatch(x)
        cdev = counts.to(xrows.device)
        recv_counts = c.all_to_all_counts(cdev).cpu().numpy()
        recv_rows = recv_counts.sum(axis=1)
        pend.recv_rows = recv_rows
        xrecv = c.all_to_all_rows(xrows, pend.send_rows, recv_rows)
        erecv = c.all_to_all_rows(erows, pend.send_rows, recv_rows)
        y, _ = self.phase_experts(recv_counts, xrecv, erecv)
        yback = c.all_to_all_rows(y, recv_rows, pend.send_rows)
        return self.phase_combine(pend, yback, out=out)


def emulate_forward(layers: list, xs: list):
    """Step W ranks' EPLayers through the phases in one process (one GPU or
    CPU), moving rows between them with plain tensor slicing: the exchange
    the NCCL path performs, without kernels that wait on one another."""
    import torch
    W = len(layers)
    st = [l.phase_dispatch(x) for l, x in zip(layers, xs)]
    counts = [s[3].numpy() for s in st]
    # recv_counts[d][s] = counts[s][d]
    ys = []
    for d in range(W):
        rc = np.stack([counts[s][d] for s in range(W)])
        xparts, eparts = [], []
        for s in range(W):
            off = int(st[s][0].send_rows[:d].sum())
            n = int(st[s][0].send_rows[d])
            xparts.append(st[s][1][off:off + n])
            eparts.append(st[s][2][off:off + n])
        y, per_src = layers[d].phase_experts(rc, torch.cat(xparts), torch.cat(eparts))
        ys.append((y, per_src))
    outs = []
    for s in range(W):
        parts = []
        for d in range(W):
            y, per_src = ys[d]
            off = int(per_src[:s].sum())
            parts.append(y[off:off + int(per_src[s])])
        outs.append(layers[s].phase_combine(st[s][0], torch.cat(parts)))
    return outs


def emulate_forward_slab(layers: list, xs: list):
    """emulate_forward for the fixed-capacity (slab) path: the same exchange with
    equal splits, moved by tensor slicing in one process."""
    import torch
    W = len(layers)
    C = layers[0].slab
    st = [l.slab_dispatch(x) for l, x in zip(layers, xs)]
    ys = []
    for d in range(W):
        recv = torch.cat([st[s][1][d * C:(d + 1) * C] for s in range(W)])
        rc = torch.stack([st[s][2][d] for s in range(W)])
        ys.append(layers[d].stages.ep_expert_rows_slab(recv, W, C, rc, layers[d].path))
    outs = []
    for s in range(W):
        yback = torch.cat([ys[d][s * C:(s + 1) * C] for d in range(W)])
        pend, idx = st[s][0], st[s][3]
        inv_slab = idx[pend.inv.to(idx.device).long()].to(torch.int32)
        outs.append(layers[s].stages.ep_combine(pend.x, yback, inv_slab, pend.gates, layers[s].path))
    return outs
