"""Worker bodies of tests/test_dist_gloo.py (module-level so torch.multiprocessing.spawn can
pickle them).  Each runs in its own process of a world-size-2 gloo group on 127.0.0.1."""
from __future__ import annotations

import os

import numpy as np
import torch
import torch.distributed as dist


def _init(rank: int, world: int, port: int) -> None:
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


def host_plumbing(rank: int, world: int, port: int) -> None:
    """shard bounds, id broadcast and max-over-ranks of paper_1803_06058_b200.dist."""
    from paper_1803_06058_b200 import dist as D
    _init(rank, world, port)
    try:
        lo, hi = D.shard_bounds(1_000_003, rank, world)
        got = torch.tensor([lo, hi], dtype=torch.int64)
        allb = [torch.zeros(2, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(allb, got)
        bounds = [tuple(int(v) for v in b) for b in allb]
        assert bounds[0][0] == 0 and bounds[-1][1] == 1_000_003
        assert all(bounds[i][1] == bounds[i + 1][0] for i in range(world - 1))
        ident = D.nccl_id_for_group(make_id=lambda: bytes(range(128)))
        assert ident == bytes(range(128))
        t = D.max_over_ranks(1.5 + rank)
        assert t == 1.5 + (world - 1)
        assert D.sum_over_ranks(1.0) == float(world)
    finally:
        dist.destroy_process_group()


def sharded_lanczos(rank: int, world: int, port: int, kind: str, passes: int, one_sync: bool = False) -> None:
    """The exchange schedule liblove runs on N GPUs, with gloo all-reduces in
    place of NCCL: each rank owns a contiguous shard of the training points; per step
      u = allreduce(W_r q_r); z = K_UU u; r_r = W_r^T z + s2 q_r; alpha = allreduce(q_r.r_r)
      r'_r = r_r - alpha q_j - beta q_{j-1}; [passes x] c = allreduce(Q_r^T r'_r), r' -= Q_r c
      beta^2 = allreduce(||r'_r||^2)
    then Rc = K_UU allreduce(W_r Q_r) L^{-T} and the mean cache.  Must equal the unsharded
    fp64 oracle (same reorthogonalisation) to round-off."""
    import oracle as O
    from paper_1803_06058_b200 import dist as D
    from synth import make_inputs, scaled_config, tiny_problem
    _init(rank, world, port)
    try:
        if kind == "cfg1":
            p = scaled_config(1)
            inp = make_inputs(p)
        else:
            p, inp = tiny_problem(kind)
        full = O.build_model(inp.X, inp.y, p.m, p.lo, p.h, p.lengthscale, p.outputscale, p.sigma2)
        k = min(p.k, 60)
        ref = O.love_precompute(full, k, reorth_passes=passes)
        lo, hi = D.shard_bounds(full.n, rank, world)
        idx, w, y = full.idx[lo:hi], full.w[lo:hi], full.y[lo:hi]
        M = full.m_total

        def allreduce(a):
            t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))
            dist.all_reduce(t)
            return t.numpy()

        Q = np.zeros((hi - lo, k))
        bn = float(np.sqrt(allreduce(np.array([y @ y]))[0]))
        Q[:, 0] = y / bn
        alpha, beta = [], []
        k_eff = k
        for j in range(k):
            u = allreduce(O.W_apply(idx, w, Q[:, j], M))
            z = O.kuu_matvec(full.cols, full.outputscale, u)
            r = O.WT_apply(idx, w, z) + full.sigma2 * Q[:, j]
            if one_sync:
                # one all-reduce of Q_j^T [r, q_j, q_{j-1}]: alpha = (Q^T r)_j,
                # Q_j^T r' = Q^T r - alpha Q^T q_j - beta Q^T q_{j-1}
                qm1 = Q[:, j - 1] if j > 0 else np.zeros(hi - lo)
                D3 = allreduce(np.stack([Q[:, :j + 1].T @ r, Q[:, :j + 1].T @ Q[:, j], Q[:, :j + 1].T @ qm1]))
                a = float(D3[0, j])
                alpha.append(a)
                if j == k - 1:
                    break
                bj = beta[j - 1] if j > 0 else 0.0
                c = D3[0] - a * D3[1] - bj * D3[2]
                r = r - a * Q[:, j] - bj * qm1 - Q[:, :j + 1] @ c
            else:
                a = float(allreduce(np.array([Q[:, j] @ r]))[0])
                alpha.append(a)
                if j == k - 1:
                    break
                r = r - a * Q[:, j] - (beta[j - 1] * Q[:, j - 1] if j > 0 else 0.0)
                for _ in range(passes):
                    c = allreduce(Q[:, :j + 1].T @ r)
                    r = r - Q[:, :j + 1] @ c
            b = float(np.sqrt(allreduce(np.array([r @ r]))[0]))
            if b < 1e-10 * (max(abs(x) for x in alpha) + 2.0 * max(beta + [b])):
                k_eff = j + 1
                break
            beta.append(b)
            Q[:, j + 1] = r / b
        assert k_eff == ref.lanczos.k_eff, (k_eff, ref.lanczos.k_eff)
        np.testing.assert_allclose(alpha[:k_eff], ref.lanczos.alpha, rtol=1e-9)
        nb = min(len(beta), k_eff - 1)
        # betas near breakdown are O(1e-8) and set by round-off of the summation order
        # (SURVEY X2): absolute bound relative to the largest beta
        np.testing.assert_allclose(beta[:nb], ref.lanczos.beta[:nb], rtol=1e-7, atol=1e-10 * max(beta))
        # replicated cache: Z = K_UU (sum_r W_r Q_r), R = Z^T, R' = T^{-1} R
        WQ = allreduce(np.stack([O.W_apply(idx, w, Q[:, i], M) for i in range(k_eff)], 1))
        Z = O.kuu_matvec(full.cols, full.outputscale, WQ)
        Ld, Ls = O.tridiag_cholesky(np.array(alpha[:k_eff]), np.array(beta[:k_eff - 1]))
        R = Z.T
        Rp = O.tridiag_solve(Ld, Ls, R)
        e1 = np.zeros(k_eff)
        e1[0] = 1.0
        a_mean = bn * (R.T @ O.tridiag_solve(Ld, Ls, e1))
        sh = O.LoveCache(R, Rp, a_mean, ref.lanczos, Ld, Ls, "y")
        Xs = inp.Xs[:200]
        v_sh, v_ref = O.predict_var(full, sh, Xs), O.predict_var(full, ref, Xs)
        np.testing.assert_allclose(v_sh, v_ref, rtol=1e-8, atol=1e-13)
        np.testing.assert_allclose(O.predict_mean(full, sh, Xs), O.predict_mean(full, ref, Xs),
                                   rtol=1e-8, atol=1e-10)
    finally:
        dist.destroy_process_group()


def liblove_host_plumbing(rank: int, world: int, port: int) -> None:
    """liblove's own host side of the N > 1 path, over gloo: rank 0 makes the NCCL unique id
    with love_nccl_unique_id (liblove.so dlopens NCCL; no GPU needed) and the caller's process
    group broadcasts it (dist.nccl_id_for_group's default); bench.py's strong-scaling shards of
    one global draw tile the training and test sets exactly, its weak-scaling shards are
    distinct draws, and both arms' `config` records agree."""
    import bench
    from paper_1803_06058_b200 import dist as D
    from synth import get_config, make_inputs
    _init(rank, world, port)
    try:
        ident = D.nccl_id_for_group()                       # love_nccl_unique_id on rank 0
        allid = [None] * world
        dist.all_gather_object(allid, ident)
        assert len(ident) == 128 and all(x == ident for x in allid) and any(ident)
        p = dataclass_replace(get_config(4), n=10_007, t=5_003)
        g = make_inputs(p)
        sh = bench.shard_inputs(p, rank, world, "strong")
        parts = [None] * world
        dist.all_gather_object(parts, (sh.X, sh.y, sh.Xs))
        np.testing.assert_array_equal(np.concatenate([q[0] for q in parts]), g.X)
        np.testing.assert_array_equal(np.concatenate([q[1] for q in parts]), g.y)
        np.testing.assert_array_equal(np.concatenate([q[2] for q in parts]), g.Xs)
        w = bench.shard_inputs(p, rank, world, "weak")
        assert len(w.X) == p.n and len(w.Xs) == p.t
        allw = [None] * world
        dist.all_gather_object(allw, w.y[:8])
        assert not np.allclose(allw[0], allw[1])             # independent shards per rank
        assert bench.config_record(p, world, "strong")["n"] == p.n
        assert bench.config_record(p, world, "weak")["n"] == world * p.n
        assert D.sum_over_ranks(float(len(sh.Xs))) == p.t
    finally:
        dist.destroy_process_group()


def dataclass_replace(p, **kw):
    import dataclasses
    return dataclasses.replace(p, **kw)
