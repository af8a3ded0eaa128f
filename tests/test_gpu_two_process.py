"""Two ranks (two processes, one device, gloo carrying the CUDA tensors) through
distributed.exchange_sharded with the native kernels: the N-rank K must be bitwise the
single-device K, with the dense int64 all-reduce and with the block-sparse one, for the
hashed and the cost-balanced plans.  The ranks' kernels never wait on one another (each
rank builds its own shard; the only exchange is the all-reduce, staged through the host
by gloo), so sharing one GPU is safe."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _setup():
    import paper_1401_6961_b200 as hx
    from paper_1401_6961_b200 import configs
    cfg = configs.cube_cluster(24, 5, "tiny")
    part = hx.build_partition(cfg.system, leaf_size=cfg.leaf_size)
    pairs = hx.build_pair_tree(cfg.system, part, tau_ovlp=cfg.tau_ovlp)
    dev = torch.device("cuda", 0)
    P = torch.from_numpy(cfg.P).to(dev)
    return hx, cfg, part, pairs, P, dev


def _worker(rank, world, port, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1401_6961_b200 import distributed
    hx, cfg, part, pairs, P, dev = _setup()
    n = cfg.n_functions
    res = {}
    for sym, tag in ((True, "fourfold"), (False, "naive")):
        for strategy in ("hashed", "balanced"):
            for sparse in (None, 64):
                Pt = hx.build_matrix_tree(P, part)
                K = torch.empty((n, n), dtype=torch.float64, device=dev)
                shards = distributed.plan(pairs, pairs, Pt, cfg.tau_2e, "schwarz", sym, world,
                                          min_tasks_per_rank=8, strategy=strategy, K_scratch=K,
                                          groups_per_rank=4)
                c, _ = distributed.exchange_sharded(pairs, pairs, Pt, cfg.tau_2e, "schwarz", sym, K,
                                                    shards=shards, sparse_block=sparse)
                torch.cuda.synchronize()
                res[f"{tag}_{strategy}_{sparse}"] = K.cpu().numpy()
                res[f"{tag}_{strategy}_{sparse}_q"] = np.int64(c.eri_shell_quartets)
    # row-owning reduce-scatter over the K quadtree (every rank saves its own rows)
    for sym, tag in ((True, "fourfold"), (False, "naive")):
        Pt = hx.build_matrix_tree(P, part)
        K = torch.empty((n, n), dtype=torch.float64, device=dev)
        shards = distributed.plan(pairs, pairs, Pt, cfg.tau_2e, "schwarz", sym, world,
                                  min_tasks_per_rank=8, strategy="hashed")
        block, tree, c, stats = distributed.exchange_sharded_rows(pairs, pairs, Pt, cfg.tau_2e, "schwarz", sym, K,
                                                                  shards=shards)
        torch.cuda.synchronize()
        np.savez(out_path + f".rows_{tag}_{rank}.npz", rows=block.dense().cpu().numpy(), f0=block.f0, f1=block.f1,
                 q=np.int64(c.eri_shell_quartets), nnz=tree.nnz_tiles, tiles=stats["leaf_tiles"],
                 packed=stats["bytes_packed"], dense=stats["bytes_dense"])
    if rank == 0:
        np.savez(out_path, **res)
    dist.barrier()
    dist.destroy_process_group()


def test_two_ranks_on_one_device_reproduce_the_single_device_K(tmp_path):
    out = str(tmp_path / "two.npz")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    res = np.load(out)
    hx, cfg, part, pairs, P, dev = _setup()
    from paper_1401_6961_b200 import exchange
    n = cfg.n_functions
    for sym, tag in ((True, "fourfold"), (False, "naive")):
        Pt = hx.build_matrix_tree(P, part)
        K1 = torch.empty((n, n), dtype=torch.float64, device=dev)
        _, c1, _ = exchange.run_exchange(pairs, pairs, Pt, cfg.tau_2e, "schwarz", sym, True, None, K_out=K1)
        K1 = K1.cpu().numpy()
        for strategy in ("hashed", "balanced"):
            for sparse in (None, 64):
                key = f"{tag}_{strategy}_{sparse}"
                assert np.array_equal(res[key], K1), key           # bitwise: exact integer all-reduce
                assert int(res[key + "_q"]) == c1.eri_shell_quartets, key
        # reduce-scatter: the two ranks' row blocks tile K; fourfold rows are (A + A^T) / 2 formed
        # in fixed point (one rounding) against the epilogue's FP64 average of two rounded values
        got = [np.load(out + f".rows_{tag}_{r}.npz") for r in range(2)]
        assert int(got[0]["f0"]) == 0 and int(got[0]["f1"]) == int(got[1]["f0"]) and int(got[1]["f1"]) == n
        Krs = np.concatenate([g["rows"] for g in got], axis=0)
        tol = 4e-16 * np.abs(K1).max() if sym else 0.0
        assert np.abs(Krs - K1).max() <= tol, tag
        assert int(got[0]["q"]) == c1.eri_shell_quartets
        assert 0 < int(got[0]["nnz"]) <= int(got[0]["tiles"])
        assert int(got[0]["packed"]) <= int(got[0]["dense"])
