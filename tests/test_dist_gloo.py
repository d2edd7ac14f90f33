"""World-size-2 gloo tests of the N > 1 path on CPU: the host-side plumbing
(shard bounds, NCCL-id broadcast, max over ranks) and the per-step exchange schedule of the
sharded Lanczos loop, which must reproduce the unsharded oracle."""
import socket

import pytest
import torch.multiprocessing as mp

import _dist_workers as W


def _port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_host_plumbing_world2():
    mp.spawn(W.host_plumbing, args=(2, _port()), nprocs=2, join=True)


@pytest.mark.parametrize("kind,passes", [("cfg1", 2), ("1d_n200", 1), ("2d", 2), ("3d", 2)])
def test_sharded_lanczos_matches_oracle_world2(kind, passes):
    mp.spawn(W.sharded_lanczos, args=(2, _port(), kind, passes), nprocs=2, join=True)


def test_liblove_host_plumbing_world2():
    mp.spawn(W.liblove_host_plumbing, args=(2, _port()), nprocs=2, join=True)


@pytest.mark.parametrize("kind", ["cfg1", "2d"])
def test_one_sync_schedule_matches_oracle_world2(kind):
    """The one-sync step liblove runs on several GPUs in fp32 (three collectives per step:
    u, the dot vectors Q_j^T [r, q_j, q_{j-1}], beta^2), in fp64 oracle arithmetic, sharded
    over 2 gloo ranks: the same Lanczos as the unsharded CGS oracle."""
    mp.spawn(W.sharded_lanczos, args=(2, _port(), kind, 1, True), nprocs=2, join=True)
