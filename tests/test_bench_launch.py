"""bench.py's launch contract on CPU (no GPU needed): `--gpus N` without a
launcher re-runs itself under torch.distributed.run with N ranks and only
rank 0 prints the JSON line; under a launcher WORLD_SIZE must equal --gpus.
Exercised through the reference arm (the CPU oracle), with a tiny time
budget (PGA_REF_BUDGET_S)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env_extra):
    env = dict(os.environ, PGA_REF_BUDGET_S="4", **env_extra)
    env.pop("WORLD_SIZE", None) if "WORLD_SIZE" not in env_extra else None
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, cwd=ROOT, env=env,
                          capture_output=True, text=True, timeout=600)


def test_gpus_flag_spawns_ranks_and_rank0_prints_one_line():
    r = _run(["--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "3"], {})
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
    assert d["cpu_baseline"]["cores"] >= 1 and "cpu_model" in d["cpu_baseline"]


def test_world_size_must_match_gpus():
    r = _run(["--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "3"],
             {"WORLD_SIZE": "1", "RANK": "0", "LOCAL_RANK": "0"})
    assert r.returncode == 2
    assert "WORLD_SIZE=1 but --gpus 2" in r.stderr
