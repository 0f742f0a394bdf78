"""Multi-process (world_size 2, gloo, CPU) test of the instance sharding and
the final gather — the only multi-GPU logic of the batched path (BASELINE
configs[2]); the per-instance march itself is the CPU oracle here."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_2002_11978_b200 import workloads as WL

N_INST, n, M = 5, 63, 6


def _march(b0, B):
    x, kx, fx, u0 = WL.instance_fields(n, b0, B)
    out = []
    for i in range(B):
        rec = O.fids_march(0.5, 1.5, 1.0, 1.0, M, 3.0, n + 1,
                           lambda xx, t, i=i: kx[i] * WL.kappa_t(t),
                           lambda xx, t, i=i: fx[i] * WL.source_t(t),
                           lambda xx, i=i: u0[i], epsilon=1e-10, tol=1e-10,
                           keep_history=False)
        out.append(rec.hist)
    return np.array(out)


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        b0, b1 = WL.shard_range(N_INST, world, rank)
        local = torch.from_numpy(_march(b0, b1 - b0))
        full = WL.gather_rows(local)
        if rank == 0:
            q.put(full.numpy())
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_ranges_partition():
    for B in (1, 5, 4096):
        for world in (1, 2, 3, 8):
            got = [WL.shard_range(B, world, r) for r in range(world)]
            assert got[0][0] == 0 and got[-1][1] == B
            assert all(a[1] == b[0] for a, b in zip(got, got[1:]))
            sizes = [b - a for a, b in got]
            assert max(sizes) - min(sizes) <= 1


def test_instance_fields_independent_of_sharding():
    _, k_all, f_all, u_all = WL.instance_fields(32, 0, 6)
    _, k_b, f_b, u_b = WL.instance_fields(32, 3, 3)
    np.testing.assert_array_equal(k_all[3:], k_b)
    np.testing.assert_array_equal(f_all[3:], f_b)
    np.testing.assert_array_equal(u_all[3:], u_b)


def test_cfg3_copy_scales_independent_of_sharding():
    all8 = WL.copy_scales(0, 8)
    assert np.all((all8 >= 0.5) & (all8 <= 2.0)) and np.unique(all8).size == 8
    for r in range(8):   # one copy per rank over 8 GPUs == the batched 8 copies
        np.testing.assert_array_equal(WL.copy_scales(r, 1), all8[r:r + 1])


def test_two_rank_gloo_shard_and_gather_matches_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    mp.start_processes(_worker, args=(2, port, q), nprocs=2, join=True, start_method="spawn")
    gathered = q.get()
    ref = _march(0, N_INST)
    assert gathered.shape == (N_INST, n)
    np.testing.assert_array_equal(gathered, ref)
