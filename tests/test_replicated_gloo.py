"""Replicated master-slave on CPU: world_size 2 and 3
processes (gloo) run paper_1403_4099_b200.replicated.ReplicatedRunner with
oracle-backed replicas.  Each rank evaluates only its shard; after the
all-gather every replica must hold the single-population run of orc_run
(n_islands = 1), generation for generation."""
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


def _worker(rank, world, port, out_path, P, gens):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    import oracle as orc
    import workloads
    from oracle_island import OracleReplica
    from paper_1403_4099_b200.replicated import ReplicatedRunner
    dist.init_process_group("gloo", rank=rank, world_size=world)
    X, _ = workloads.noh_returns(workloads.CONFIGS["C1"])
    C = orc.pearson(X)
    eng = OracleReplica(C, orc.default_params(pop=P, max_gens=gens, tol=-1.0, seed=5))
    runner = ReplicatedRunner(eng)
    eng.init(5)
    runner.run(gens)
    res = {"history": eng.history, "best_L": eng.best_ever, "best": eng.best_labels.tolist(),
           "evaluated": eng.evaluated, "shard": [runner.begin, runner.end],
           "pop": eng.pop.tolist()}
    json.dump(res, open(out_path % rank, "w"))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,P", [(2, 100), (3, 130)])
def test_replicated_gloo_matches_single_population(tmp_path, world, P):
    import oracle as orc
    import workloads
    gens = 9
    out = str(tmp_path / "r%d.json")
    mp.start_processes(_worker, args=(world, _free_port(), out, P, gens), nprocs=world, join=True,
                       start_method="spawn")
    X, _ = workloads.noh_returns(workloads.CONFIGS["C1"])
    C = orc.pearson(X)
    ref = orc.run(C, orc.default_params(pop=P, max_gens=gens, tol=-1.0, seed=5))
    res = [json.load(open(out % r)) for r in range(world)]
    covered = []
    for r in res:
        assert np.array_equal(np.array(r["history"]), ref["history"])
        assert r["best_L"] == ref["best_L"]
        assert np.array_equal(np.array(r["best"]), ref["best_labels"])
        assert r["pop"] == res[0]["pop"]                  # replicas identical
        b, e = r["shard"]
        assert b % 32 == 0
        assert r["evaluated"] == (e - b) * gens           # each rank evaluated only its shard
        covered += list(range(b, e))
    assert sorted(covered) == list(range(P))              # shards partition the population
