"""Expert-parallel orchestration on CPU: world_size 2 (and 3) over gloo.

The exchange logic of paper_2605_09281_b200/ep.py (count matrix, split
sizes, segment construction, return path, combine order) runs unchanged; the
per-rank compute stages are checker-backed (oracle/), so each rank's output
must equal the single-process oracle tileq_forward on its own tokens.
SURVEY.md §8(e).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import REPO, rel_frob

SPEC = dict(K=6, top_k=2, i=256, o=192, S=1, bits=3, r=8, group=128, tier="general", seed=7)


class OracleStages:
    """The Layer stage interface (route / permute / ep_*) backed by the C oracle,
    for the rank owning experts [e_begin, e_end).  Rows are f32 token rows; the
    extension row carries the (token, slot) so transport is checked too."""

    def __init__(self, oracle, art, e_begin, e_end):
        self.o, self.art = oracle, art
        self.num_experts, self.top_k = art["K"], art["top_k"]
        self.in_dim, self.out_dim = art["i"], art["o"]
        self.e_begin, self.e_end = e_begin, e_end
        self.single = dict(art, top_k=1, shared=[], S=0)

    def route(self, x):
        ids, gates = self.o.route(x.numpy(), self.art["gate"], self.top_k)
        return torch.from_numpy(ids.astype(np.int32)), torch.from_numpy(gates)

    def permute(self, ids):
        p, off, inv = self.o.permute(ids.numpy().astype(np.int64), self.num_experts)
        return torch.from_numpy(p), torch.from_numpy(off), torch.from_numpy(inv)

    def ep_dispatch_rows(self, x, ids, perm, path):
        tok = perm.long() // self.top_k
        xrows = x[tok].clone()
        erows = torch.stack([tok.float(), ids.reshape(-1)[perm.long()].float()], 1)
        return xrows, erows

    def ep_expert_rows(self, xrows, erows, segs, path):
        y = torch.zeros((xrows.shape[0], self.out_dim), dtype=torch.float32)
        for j, r0, n in segs:
            e = self.e_begin + int(j)
            assert e < self.e_end
            # the expert id travelled with the row: it must be the segment's expert
            assert (erows[r0:r0 + n, 1] == e).all()
            xs = xrows[r0:r0 + n].numpy()
            ids = np.full((n, 1), e, np.int64)
            g1 = np.ones((n, 1), np.float32)
            a = self.o.qmoe_forward(self.single, xs, ids, g1)
            b = self.o.lotile_forward(self.single, xs, ids, g1)
            y[r0:r0 + n] = torch.from_numpy(a.astype(np.float64) + b)
        return y

    def ep_expert_rows_slab(self, rows, n_src, slab, counts, path):
        # the checker's rows are [x (in_dim f32) | (token, expert)]: split, rebuild the
        # (source, expert) segments from the received counts, reuse ep_expert_rows
        xw = self.in_dim
        cnt = counts.numpy()
        segs = []
        for s in range(n_src):
            r = s * slab
            for j in range(cnt.shape[1]):
                if self.e_begin + j < self.e_end and cnt[s, j]:
                    segs.append((j, r, int(cnt[s, j])))
                r += int(cnt[s, j])
        return self.ep_expert_rows(rows[:, :xw], rows[:, xw:], segs, path)

    def ep_combine(self, x, yrows, inv, gates, path, out=None):
        B = x.shape[0]
        k = self.top_k
        Y = yrows.double()[inv.long()].reshape(B, k, self.out_dim)
        acc = (gates.double().unsqueeze(-1) * Y).sum(1)
        if self.art["S"]:
            ids0 = np.zeros((B, k), np.int64)
            acc += torch.from_numpy(self.o.qmoe_forward(self.art, x.numpy(), ids0, np.zeros((B, k), np.float32))).double()
        y = acc.float()
        if out is not None:
            out.copy_(y)
            return out
        return y


def _art(tmpdir):
    from paper_2605_09281_b200 import synth
    d = os.path.join(tmpdir, "ep_art")
    if not os.path.exists(os.path.join(d, "manifest.json")):
        synth.write_synthetic(d, **SPEC)
    return d


def _worker(rank, world, port, art_dir, batches, q, slab=None):
    import sys
    sys.path.insert(0, REPO)
    sys.path.insert(0, os.path.join(REPO, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.oracle import Oracle, read_artifact_np
        from paper_2605_09281_b200.ep import EPLayer, TorchComm
        o = Oracle()
        art = read_artifact_np(art_dir)
        comm = TorchComm()
        from paper_2605_09281_b200.ep import expert_bounds
        b = expert_bounds(art["K"], world)
        ep = EPLayer(comm=comm, stages=OracleStages(o, art, b[rank], b[rank + 1]), slab=slab)
        errs = []
        for B in batches:
            # ranks hold different token counts (ragged, including empty)
            Br = (B + 3 * rank if B else 0) if slab is None else B
            x = np.random.default_rng(1000 * rank + B).standard_normal((Br, art["i"])).astype(np.float32)
            y = ep.forward(torch.from_numpy(x)).numpy()
            want = o.tileq_forward(art, x)[0] if Br else np.zeros((0, art["o"]), np.float32)
            errs.append((Br, rel_frob(y, want) if Br else 0.0, y.shape == want.shape))
        q.put((rank, errs))
    except Exception as e:  # report instead of hanging the peer
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.fixture(scope="module")
def oracle_built(oracle):
    return oracle


@pytest.mark.parametrize("world", [2, 3])
def test_ep_gloo_matches_oracle(oracle_built, tmp_path_factory, world):
    art_dir = _art(str(tmp_path_factory.mktemp("ep")))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, art_dir, [1, 5, 0, 40], q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    for r in range(world):
        assert not isinstance(res[r], str), res[r]
        for Br, err, shape_ok in res[r]:
            assert shape_ok
            assert err <= 1e-5, (r, Br, err)


@pytest.mark.parametrize("world", [2, 3])
def test_ep_gloo_slab_matches_oracle(oracle_built, tmp_path_factory, world):
    """Fixed-capacity (slab) exchange: equal-split all-to-alls, receive-side
    segments from the exchanged count matrix -- no host round trip on GPUs."""
    art_dir = _art(str(tmp_path_factory.mktemp("ep_slab")))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, art_dir, [1, 5, 16], q, 40)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    for r in range(world):
        assert not isinstance(res[r], str), res[r]
        for Br, err, shape_ok in res[r]:
            assert shape_ok
            assert err <= 1e-5, (r, Br, err)


def test_send_plan_and_segments():
    from paper_2605_09281_b200.ep import expert_bounds, recv_segments, send_plan
    b = expert_bounds(60, 8)
    assert b[0] == 0 and b[-1] == 60 and all(b[r + 1] - b[r] in (7, 8) for r in range(8))
    offs = np.cumsum([0] + [3, 0, 2, 5, 1, 4])
    rows, counts = send_plan(offs, expert_bounds(6, 2))
    assert rows.tolist() == [5, 10]
    assert counts.tolist() == [[3, 0, 2], [5, 1, 4]]
    per_src, segs = recv_segments(np.array([[3, 0, 2], [1, 1, 0]]), 3)
    assert per_src.tolist() == [5, 2]
    assert segs.tolist() == [[0, 0, 3], [2, 3, 2], [0, 5, 1], [1, 6, 1]]
    with pytest.raises(Exception):
        expert_bounds(2, 4)
