"""world_size-2 gloo tests of the N>1 path on CPU: contiguous sharding covers
every realization once, and the final all-gather returns results in global
order, identical to a single-process solve (the reference's parallel ==
serial invariant, test_harness.py:144-154).  The per-shard solve is the CPU
oracle here (no GPU in this container); on a GPU box the same code calls the
CUDA engine."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2510_20507_b200.sharding import GATHER_FIELDS, shard_bounds


def test_shard_bounds_cover_exactly_once():
    for total in (1, 2, 7, 64, 1000):
        for world in (1, 2, 3, 8):
            seen = []
            for r in range(world):
                s, e = shard_bounds(total, world, r)
                seen.extend(range(s, e))
            assert seen == list(range(total))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _oracle_solve(b):
    from oracle import ammmse_oracle as orc
    from paper_2510_20507_b200.solvers import BatchResult

    r = orc.solve_batch(b.channels, b.noise_power, b.weights, b.p_max, b.init_precoders, 0.01, 0.5,
                        eps2=1e-4, max_iters=40)
    return BatchResult(r["final_precoders"], r["wsr_bits"], r["iterations"],
                       r["converged"].astype(np.uint8), r["stationarity_residual"],
                       r["switch_iteration"], r["status"], r["gamma_used"])


def _worker(rank, world, port, out_path):
    import torch.distributed as dist

    from paper_2510_20507_b200.inputs import build_batch
    from paper_2510_20507_b200.sharding import solve_sharded

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    b = build_batch(8, 2, 2, 1, 5, p_max=4.0, dtype=np.complex128)
    res, _ = solve_sharded(b, None, solve_fn=_oracle_solve)
    if rank == 0:
        np.savez(out_path, **res)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gather_equals_serial(tmp_path):
    from paper_2510_20507_b200.inputs import build_batch
    from paper_2510_20507_b200.sharding import pack_scalars, unpack_scalars

    out = str(tmp_path / "res.npz")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    got = np.load(out)
    serial = unpack_scalars(pack_scalars(_oracle_solve(build_batch(8, 2, 2, 1, 5, p_max=4.0,
                                                                   dtype=np.complex128))))
    for f in GATHER_FIELDS:
        assert np.array_equal(got[f], serial[f]), f
