"""World-size-2 and -4 model of the multi-GPU path on CPU (gloo): rows
sharded with paper_2603_11953_b200.sharding, rank-local partial Grams (the
restatement stands in for the device kernel), ONE exchange as Plan::exchange
does it (engine.cu): an all-gather of every rank's partial, then the
reference's fixed tree over ranks (parallel_gram.cpp:93-102) with binary64
adds for fp64 and dd_add for double-double (a plain sum would drop the lo
words); redundant Jacobi identical on every rank, and rank-local U rows that
concatenate to the single-process U. The device side of the combine is
pinned bitwise to the same tree by tests/test_configs_gpu.py
(mpsvd_stage_rank_combine)."""
from __future__ import annotations

import os
import socket
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _matrix(m, n, dtype, seed=5):
    r = np.random.default_rng(seed)
    b = r.standard_normal((n, m))
    b /= np.linalg.norm(b, axis=1)[:, None]
    d = 10.0 ** (-6.0 * np.arange(n) / (n - 1))
    return np.asfortranarray((b * d[:, None]).T.astype(dtype))


def _worker(rank, world, port, out_dir):
    sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), HERE]
    import pyoracle
    from helpers import dd_add_elementwise, rank_tree
    from paper_2603_11953_b200 import sharding

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    P = pyoracle.Port()
    m, n = 3001, 24
    r0, r1 = sharding.local_rows(m, world, rank)

    # ---- fp64 Gram of fp32 A: local partial + one all-gather + rank tree
    a32 = _matrix(m, n, np.float32)
    loc = P.partitioned_gram_f32(np.asfortranarray(a32[r0:r1]), blocks=min(16, r1 - r0))
    t = torch.from_numpy(np.ascontiguousarray(loc))
    gl = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(gl, t)
    g = rank_tree([x.numpy().copy() for x in gl], lambda x, y: x + y)
    lam, v, _, _ = P.twosided_jacobi(g, sem=pyoracle.SEM_DEVICE)
    # redundant Jacobi: identical bits on every rank
    lam_all = [torch.zeros(n, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(lam_all, torch.from_numpy(lam))
    same = all(np.array_equal(x.numpy(), lam) for x in lam_all)
    sigma = np.sqrt(lam).astype(np.float32)
    w = (v.astype(np.float32) / sigma[None, :]).astype(np.float32)
    u_loc = P.av_f32(np.asfortranarray(a32[r0:r1]), w)

    # ---- double-double Gram of fp64 A: all-gather (hi, lo) + rank-order dd sum
    a64 = _matrix(m, n, np.float64, seed=6)
    hi, lo = P.dd_gram(np.asfortranarray(a64[r0:r1]), threads=2)
    pair = torch.from_numpy(np.stack([hi, lo]))
    gath = [torch.zeros_like(pair) for _ in range(world)]
    dist.all_gather(gath, pair)
    acc_h, acc_l = rank_tree([(x[0].numpy().copy(), x[1].numpy().copy()) for x in gath],
                             lambda x, y: dd_add_elementwise(P, x, y))
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), g=g, lam=lam, same=same, u=u_loc, r0=r0, r1=r1,
             w=w, ddh=acc_h, ddl=acc_l)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
@pytest.mark.parametrize("world", [2, 4])
def test_sharded_pipeline(tmp_path, port, world):
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    res = [dict(np.load(tmp_path / f"rank{r}.npz")) for r in range(world)]
    m, n = 3001, 24
    a32 = _matrix(m, n, np.float32)
    g_full = port.partitioned_gram_f32(a32, blocks=16)
    d = np.sqrt(np.diag(g_full))
    for r in res:
        assert bool(r["same"])
        assert np.array_equal(r["g"], r["g"].T)
        # both sums within m*u_h*||a_i|| ||a_j|| of the exact Gram
        assert np.all(np.abs(r["g"] - g_full) <= 2 * m * 2.0 ** -53 * np.outer(d, d))
    for r in res[1:]:
        assert np.array_equal(res[0]["lam"], r["lam"]) and np.array_equal(res[0]["w"], r["w"])
        assert np.array_equal(res[0]["g"], r["g"])
    # rank-local U rows concatenate to the single-process U for the same W
    u = np.concatenate([r["u"] for r in res], axis=0)
    assert np.array_equal(u, port.av_f32(a32, res[0]["w"]))
    # dd: the gathered, rank-ordered compensated sum matches the single-pass dd Gram
    a64 = _matrix(m, n, np.float64, seed=6)
    hh, ll = port.dd_gram(a64, threads=4)
    an = np.linalg.norm(a64, axis=0)
    err = np.abs((res[0]["ddh"] - hh) + (res[0]["ddl"] - ll))
    assert np.all(err <= 4 * (m * 2.0 ** -53) ** 2 * np.outer(an, an) + 2.0 ** -100 * np.abs(hh))
    for r in res[1:]:
        assert np.array_equal(res[0]["ddh"], r["ddh"]) and np.array_equal(res[0]["ddl"], r["ddl"])


def _worker_ozaki(rank, world, port, out_dir):
    # K2z on the sharded path: every rank slices its own rows with its own
    # column exponents (the restatement stands in for gram_dd_ozaki), then
    # the dd exchange of the library (all-gather + rank-ordered dd_add)
    sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), HERE]
    import pyoracle
    from paper_2603_11953_b200 import sharding

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    P = pyoracle.Port()
    m, n = 10001, 20
    r0, r1 = sharding.local_rows(m, world, rank)
    a64 = _matrix(m, n, np.float64, seed=7)
    loc = np.asfortranarray(a64[r0:r1])
    nch = (r1 - r0 + 31) // 32
    scb = np.linspace(0, nch, 9).astype(np.int32)  # 8 chunk-aligned splits
    bsb = np.array([0, 2, 4, 6, 8], np.int32)       # 4 logical blocks
    hi, lo = P.gram_dd_ozaki(loc, scb, bsb, span_cap=5)
    pair = torch.from_numpy(np.stack([hi, lo]))
    gath = [torch.zeros_like(pair) for _ in range(world)]
    dist.all_gather(gath, pair)
    from helpers import dd_add_elementwise, rank_tree

    acc_h, acc_l = rank_tree([(x[0].numpy().copy(), x[1].numpy().copy()) for x in gath],
                             lambda x, y: dd_add_elementwise(P, x, y))
    np.savez(os.path.join(out_dir, f"oz{rank}.npz"), h=acc_h, l=acc_l)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_ozaki_gram_exchange(tmp_path, port):
    world = 2
    mp.start_processes(_worker_ozaki, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    res = [dict(np.load(tmp_path / f"oz{r}.npz")) for r in range(world)]
    assert np.array_equal(res[0]["h"], res[1]["h"]) and np.array_equal(res[0]["l"], res[1]["l"])
    m, n = 10001, 20
    a64 = _matrix(m, n, np.float64, seed=7)
    hh, ll = port.dd_gram(a64, threads=4)
    an = np.linalg.norm(a64, axis=0)
    err = np.abs((res[0]["h"] - hh) + (res[0]["l"] - ll)) / np.outer(an, an)
    # the K2z error level (rank-local exponents change nothing about it)
    assert err.max() <= 2.0 ** -80
    assert np.array_equal(res[0]["h"], res[0]["h"].T)
