"""The N>1 path on CPU: two processes (gloo, world_size 2) run the island
driver (paper_1403_4099_b200.islands.IslandRunner) with oracle-backed
engines; the all-gathered migrant records must reproduce the oracle's
single-process two-island simulation (orc_run with n_islands = 2)
generation for generation."""
import json
import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_path, gens, tol=-1.0, stall=50):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    import oracle as orc
    import workloads
    from oracle_island import OracleIsland
    from paper_1403_4099_b200.islands import IslandRunner
    dist.init_process_group("gloo", rank=rank, world_size=world)
    X, planted = workloads.noh_returns(workloads.CONFIGS["C1"])
    C = orc.pearson(X)
    params = orc.default_params(pop=48, max_gens=gens, tol=tol, stall_gens=stall, n_islands=world,
                                migrate_every=4, migrants=5, seed=77)
    eng = OracleIsland(C, params, rank, world)
    runner = IslandRunner(eng)
    eng.init(77)
    stepped = runner.run(gens)
    bestL, best, isl = runner.global_best()
    # per-generation global best = max over islands
    import torch
    h = torch.tensor(eng.history, dtype=torch.float64)
    parts = [torch.zeros_like(h) for _ in range(world)]
    dist.all_gather(parts, h)
    if rank == 0:
        json.dump({"history": torch.stack(parts).max(0).values.tolist(), "best_L": bestL,
                   "exchanges": runner.exchanges, "stepped": stepped,
                   "generation": eng.state()["generation"]}, open(out_path, "w"))
    dist.barrier()
    dist.destroy_process_group()


def test_two_islands_gloo_matches_oracle(tmp_path):
    import oracle as orc
    import workloads
    gens = 13
    out = str(tmp_path / "res.json")
    mp.start_processes(_worker, args=(2, _free_port(), out, gens), nprocs=2, join=True,
                       start_method="spawn")
    res = json.load(open(out))
    X, _ = workloads.noh_returns(workloads.CONFIGS["C1"])
    C = orc.pearson(X)
    ref = orc.run(C, orc.default_params(pop=48, max_gens=gens, tol=-1.0, n_islands=2,
                                        migrate_every=4, migrants=5, seed=77))
    assert res["exchanges"] == gens // 4
    assert np.array_equal(np.array(res["history"]), ref["history"])
    assert res["best_L"] == ref["best_L"]


def test_two_islands_gloo_stall_termination_matches_oracle(tmp_path):
    """Live tolerance (Q28): both ranks stop at the generation orc_run's
    two-island rule gives, with the same per-generation global best."""
    import oracle as orc
    import workloads
    gens, tol, stall = 200, 1e-5, 8
    out = str(tmp_path / "res.json")
    mp.start_processes(_worker, args=(2, _free_port(), out, gens, tol, stall), nprocs=2, join=True,
                       start_method="spawn")
    res = json.load(open(out))
    X, _ = workloads.noh_returns(workloads.CONFIGS["C1"])
    C = orc.pearson(X)
    ref = orc.run(C, orc.default_params(pop=48, max_gens=gens, tol=tol, stall_gens=stall, n_islands=2,
                                        migrate_every=4, migrants=5, seed=77))
    assert ref["reason"] == 1 and ref["gens_run"] < gens
    assert res["stepped"] == ref["gens_run"]
    assert np.array_equal(np.array(res["history"]), ref["history"])
    assert res["best_L"] == ref["best_L"]
