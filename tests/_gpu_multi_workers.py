"""Worker bodies of tests/test_gpu_multi.py (module-level so torch.multiprocessing.spawn can
pickle them): one process per GPU, NCCL process group on 127.0.0.1, liblove's own sharded
build (its NCCL all-reduces of u, alpha, the reorthogonalisation dots and beta^2)."""
from __future__ import annotations

import os

import numpy as np
import torch
import torch.distributed as dist


def sharded_equals_single(rank: int, world: int, port: int, ci: int, n: int, m, k: int, t: int,
                          out_dir: str) -> None:
    from paper_1803_06058_b200 import LoveCache, nccl_unique_id
    from paper_1803_06058_b200 import dist as D
    from synth import make_inputs, scaled_config
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    try:
        p = scaled_config(ci, n=n, m=m, k=k, t=t)
        g = make_inputs(p)
        lo, hi = D.shard_bounds(p.n, rank, world)
        ident = D.nccl_id_for_group(make_id=nccl_unique_id)
        c = LoveCache.build(g.X[lo:hi], g.y[lo:hi], p.m, p.lo, p.h, p.lengthscale, p.outputscale, p.sigma2,
                            p.k, precision=p.precision, rank=rank, world=world, nccl_id=ident)
        info = c.info()
        assert info["n_global"] == p.n and info["n_local"] == hi - lo
        var, mean = c.predict_var(g.Xs, return_mean=True)
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), var=var.double().cpu().numpy(),
                 mean=mean.double().cpu().numpy(), alpha=info["alpha"], beta=info["beta"],
                 k_eff=info["k_eff"])
        c.free()
    finally:
        dist.destroy_process_group()
