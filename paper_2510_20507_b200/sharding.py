"""Data-parallel sharding of realizations across GPUs.

Realizations are independent, so a batch shards into contiguous blocks of
ceil(B / world) global indices with no traffic during the solve; seeds are
by global index, so results do not depend on the GPU count (the reference's
own "parallel == serial" invariant, harness.py:482-490 / test_harness.py:144-154).
The only collective is the final all-gather of the per-realization result
fields, in global realization order.
"""

from __future__ import annotations

import numpy as np

# per-realization scalar fields gathered after a sharded solve
GATHER_FIELDS = ("wsr_bits", "iterations", "converged", "stationarity_residual",
                 "switch_iteration", "status", "gamma_used")


def shard_bounds(total: int, world: int, rank: int) -> tuple[int, int]:
    """[start, stop) of rank's contiguous block; blocks are ceil(total/world)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError(f"bad rank {rank} of world {world}")
    per = -(-total // world)
    start = min(total, rank * per)
    return start, min(total, start + per)


def pack_scalars(res) -> np.ndarray:
    """(B, len(GATHER_FIELDS)) float64 matrix of a host BatchResult."""
    cols = [np.asarray(getattr(res, f), dtype=np.float64) for f in GATHER_FIELDS]
    return np.stack(cols, axis=1) if cols[0].size else np.zeros((0, len(GATHER_FIELDS)))


def unpack_scalars(mat: np.ndarray) -> dict:
    out = {}
    for j, f in enumerate(GATHER_FIELDS):
        col = mat[:, j]
        if f in ("iterations", "switch_iteration", "status"):
            col = col.astype(np.int32)
        elif f == "converged":
            col = col.astype(np.uint8)
        out[f] = col
    return out


def gather_scalars(local: np.ndarray, total: int, group=None, device=None) -> np.ndarray:
    """All-gather every rank's (B_r, F) block into the global (total, F)
    matrix in realization order.  Pads ragged blocks to ceil(total/world)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    if device is None and dist.get_backend(group) == "nccl":  # NCCL gathers device tensors
        device = torch.device("cuda", torch.cuda.current_device())
    per = -(-total // world)
    F = local.shape[1]
    buf = torch.zeros((per, F), dtype=torch.float64, device=device)
    if local.shape[0]:
        buf[: local.shape[0]] = torch.from_numpy(np.ascontiguousarray(local)).to(buf.device)
    out = torch.empty((world * per, F), dtype=torch.float64, device=device)
    dist.all_gather_into_tensor(out, buf, group=group)
    return out[:total].cpu().numpy()


def solve_sharded(batch, options, snr_db: float = 10.0, device=None, solve_fn=None):
    """Solve the rank's shard of a global host Batch and gather the scalar
    results of all realizations to every rank (global order).

    ``solve_fn(shard_batch) -> BatchResult`` defaults to the CUDA engine
    (run_ammmse_batch); tests substitute the CPU oracle to exercise the
    sharding and gather logic on gloo."""
    import torch.distributed as dist

    world = dist.get_world_size() if dist.is_initialized() else 1
    rank = dist.get_rank() if dist.is_initialized() else 0
    s, e = shard_bounds(batch.B, world, rank)
    shard = batch.subset(slice(s, e))
    if solve_fn is None:
        from .solvers import run_ammmse_batch

        def solve_fn(b):
            return run_ammmse_batch(b.channels, b.noise_power, b.p_max, b.weights,
                                    b.init_precoders, options, snr_db=snr_db, device=device,
                                    step_gamma=b.gamma, step_omega=b.omega)
    local = solve_fn(shard) if e > s else None
    mat = pack_scalars(local) if local is not None else np.zeros((0, len(GATHER_FIELDS)))
    if world == 1:
        return unpack_scalars(mat), local
    return unpack_scalars(gather_scalars(mat, batch.B, device=device)), local
