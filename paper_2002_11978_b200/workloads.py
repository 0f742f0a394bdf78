"""Synthetic workloads of BASELINE.json and their multi-GPU sharding.

configs[2]: B independent instances, n = 4096, per-instance seeded fields
(SURVEY.md §8(d)):  with rng = default_rng([seed, b]) for GLOBAL instance
index b,
    g(x)   = sum_{k=1..8} a_k cos(k pi x) + b_k sin(k pi x),  a_k, b_k ~ N(0, 1/k^2)
    kappa  = exp(0.4 g(x)) * (1 + 0.2 t)
    f      = (sum_{k=1..8} c_k sin(k pi (x+1)/2)) * (1 + t),    c_k ~ N(0, 1/k^2)
    phi    = (1 - x^2)^2 * U,                                   U ~ U[0.5, 2]
configs[3] copies: when configs[3] runs as several
instances (8 seeded copies over 8 GPUs, or a batch on one), copy b is the
configs[0]-style problem with phi scaled by U_b ~ U[0.5, 2] drawn from
default_rng([seed, 3, b]) (`copy_scales`); the single-instance config keeps
U = 1.
Instances are sharded across ranks in contiguous blocks; the fields of an
instance depend only on its global index, so any sharding reproduces the
same per-instance problems (checked by tests/test_shard_gloo.py).  The time
march is sequential; instances share nothing, so the hot
path has no collective — only an optional final gather.
"""

from __future__ import annotations

import numpy as np

SEED = 2002_11978


def grid(n: int, l: float = 1.0) -> np.ndarray:
    """Interior points x_i = -l + i h, h = 2l/N, N = n + 1 (ifl.py:43-45)."""
    N = n + 1
    return -l + (2.0 * l / N) * np.arange(1, N)


def shard_range(global_batch: int, world: int, rank: int):
    """Contiguous block of global instance indices owned by `rank`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(global_batch, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def instance_fields(n: int, b0: int, B: int, seed: int = SEED):
    """Spatial parts of configs[2] for global instances b0 .. b0+B-1.

    Returns (x, kappa_x [B,n], f_x [B,n], u0 [B,n]); kappa(x,t) =
    kappa_x (1 + 0.2 t), f(x,t) = f_x (1 + t).
    """
    x = grid(n)
    k = np.arange(1, 9)
    cos_b = np.cos(np.pi * np.outer(k, x))
    sin_b = np.sin(np.pi * np.outer(k, x))
    sin_f = np.sin(np.pi * np.outer(k, (x + 1.0) / 2.0))
    A = np.empty((B, 8))
    Bc = np.empty((B, 8))
    Cc = np.empty((B, 8))
    U = np.empty(B)
    for i in range(B):
        rng = np.random.default_rng([seed, b0 + i])
        A[i] = rng.normal(0.0, 1.0 / k)
        Bc[i] = rng.normal(0.0, 1.0 / k)
        Cc[i] = rng.normal(0.0, 1.0 / k)
        U[i] = rng.uniform(0.5, 2.0)
    kx = np.exp(0.4 * (A @ cos_b + Bc @ sin_b))
    fx = Cc @ sin_f
    u0 = (1.0 - x * x) ** 2 * U[:, None]
    return x, kx, fx, u0


def copy_scales(b0: int, B: int, seed: int = SEED) -> np.ndarray:
    """U_b ~ U[0.5, 2] of the configs[3] seeded copies b0 .. b0+B-1 (global indices)."""
    return np.array([np.random.default_rng([seed, 3, b0 + i]).uniform(0.5, 2.0)
                     for i in range(B)])


def kappa_t(t: float) -> float:
    return 1.0 + 0.2 * t


def source_t(t: float) -> float:
    return 1.0 + t


def gather_rows(local, group=None):
    """All-gather a [B_local, ...] torch tensor of every rank into rank order.

    Ranks may own different counts (shard_range); the gather pads to the
    largest shard and trims.  Works with the nccl (GPU) and gloo (CPU)
    backends — this is the only collective of the multi-GPU path and it runs
    after the march, outside the timed region.
    """
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    cnt = torch.tensor([local.shape[0]], device=local.device)
    counts = [torch.zeros_like(cnt) for _ in range(world)]
    dist.all_gather(counts, cnt, group=group)
    counts = [int(c.item()) for c in counts]
    mx = max(counts)
    pad = torch.zeros((mx,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    return torch.cat([p[:c] for p, c in zip(parts, counts)], dim=0)
