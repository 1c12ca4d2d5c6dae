#!/usr/bin/env python
"""Benchmark of the B200 Giada–Marsili PGA hot path (BASELINE.json config 4).

A step is one GA generation of the whole hot path (SURVEY §8(a) a3-a11:
fitness sweep + fold, statistics/termination, isolate fittest, elitism,
scaling, SUS selection, mating, crossover, mutation, canonicalisation,
replacement; plus the elite migration all-gather every 10 generations when
N > 1) over the C4 workload: N = 500 assets, P = 65536 chromosomes in total,
sharded as islands over the ranks (strong scaling).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl pga|reference]

Prints ONE JSON line on rank 0.  `--impl reference` times the CPU oracle
(the reference arm of this tier) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads  # noqa: E402

CONFIG = "C4"            # default workload (BASELINE configs[3]); --config selects another
P_TOTAL = 65536
# population per config (BASELINE.json configs) and mutation rate (Q13)
CFG_POP = {"C1": 128, "C2": 1024, "C3": 4096, "C4": 65536, "C5": 262144}
SEED = 2024
SM_COUNT = 148
FP64_LANES_PER_SM = 64           # DFMA lanes / clk / SM (B200: 37 TF fp64 = 148*64*2*1.965G)
# SURVEY §8(d) headline ceiling for executed pair-updates: ISETP + SEL per
# pair on the 64-op/clk/SM integer/logic pipe = 32 pairs per SM-clock.
ALU_PAIRS_PER_CLK = 32
# Measured ceiling of the exact fp64 masked-accumulate inner loop on this pool
# (tools/mb_pairloop.cu, shared-memory resident, no pipeline/fold): 26.8
# executed pair-updates per SM-clock, register-file-read bound.
LOOP_PAIRS_PER_CLK = 26.8
# Measured random 8-byte gather rate from an L2-resident 2 MB fp64 array (C at
# N = 500) on this pool (tools/mb_l2gather.cu): the label-sparse pass's bound.
L2_GATHERS_PER_S = 3.03e11

METRIC = ("GA generation throughput, nominal pair-updates/s (N^2 * P per generation; "
          "fitness + all operators)")


def env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


# ---------------------------------------------------------------------------
# clocks during the timed region (B200_PROFILING.md clocks line)
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpus):
        self.gpus = gpus
        self.proc = None
        self.path = os.path.join("/tmp", "pga_clocks_%d.csv" % os.getpid())

    def start(self):
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "--query-gpu=" + self.FIELDS, "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.f.close()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                idx = int(parts[0])
            except ValueError:
                continue
            if idx not in self.gpus:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                pass
            for n, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        os.unlink(self.path)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU oracle timing (cpu_baseline and --impl reference)
# ---------------------------------------------------------------------------
def oracle_generation(orc, C, pop, params, gen):
    L, top = orc.evaluate(C, pop, nthreads=os.cpu_count() or 1)
    return orc.step(params, pop, L, top, gen)


def oracle_rate(C, planted, target_s=12.0, max_P=65536):
    """Time the oracle's full generations (evaluate on all host cores + the
    single-threaded operators) on the bench population, evolving it for as
    many generations as fit in ~target_s; plus one evaluate on a single
    thread.  Returns (nominal pair-updates/s, population, generations,
    seconds, single-thread evaluate pair-updates/s)."""
    import oracle as orc
    orc.build()
    N = C.shape[0]
    P = max_P
    pop = orc.canonicalize(workloads.population_mix(SEED, planted, P))
    params = orc.default_params(pop=P, elite=10, p_m=2.0 / N, tol=-1.0, seed=SEED)
    g, t0 = 0, time.perf_counter()
    while g == 0 or time.perf_counter() - t0 < target_s:
        pop = oracle_generation(orc, C, pop, params, g)
        g += 1
    dt = time.perf_counter() - t0
    sub = pop[:max(64, min(P, 2048))]
    t1 = time.perf_counter()
    orc.evaluate(C, sub, nthreads=1)
    d1 = time.perf_counter() - t1
    return N * N * P * g / dt, P, g, dt, N * N * sub.shape[0] / d1


def parity_probe(C, pop, L_gpu, cores, rows=4096):
    """The oracle (cpu_baseline leg) re-evaluates a sample of the GPU's last
    evaluated population: max |dL| / max(1, |L|) against north_star's 1e-9."""
    import oracle as orc
    orc.build()
    P = pop.shape[0]
    idx = np.unique(np.concatenate([np.linspace(0, P - 1, min(rows, P)).astype(np.int64), [0, P - 1]]))
    t0 = time.perf_counter()
    Lo, _ = orc.evaluate(C, pop[idx], nthreads=cores)
    dt = time.perf_counter() - t0
    err = np.abs(L_gpu[idx] - Lo) / np.maximum(1.0, np.abs(Lo))
    return {"rows": int(idx.size), "max_rel_dL": float(err.max()), "tolerance": 1e-9,
            "pass": bool(err.max() <= 1e-9), "oracle_seconds": dt,
            "what": "oracle orc_evaluate of evenly spaced rows of the GPU's last evaluated population "
                    "(labels and L read back together after the timed region)"}


def run_reference(args):
    rank = env_int("RANK", 0)
    if rank != 0:
        return 0
    import oracle as orc
    orc.build()
    X, planted = workloads.noh_returns(workloads.CONFIGS[CONFIG])
    C = orc.pearson(X)
    N = C.shape[0]
    K, W = args.steps, args.warmup
    # size each step so the whole run stays within ~3 minutes
    budget = float(os.environ.get("PGA_REF_BUDGET_S", "150")) / max(1, K + W)
    P = 256
    pop = orc.canonicalize(workloads.population_mix(SEED, planted, P))
    params = orc.default_params(pop=P, elite=10, p_m=2.0 / N, tol=-1.0, seed=SEED)
    t = time.perf_counter()
    oracle_generation(orc, C, pop, params, 0)
    dt = time.perf_counter() - t
    P = int(max(64, min(P_TOTAL, P * budget / max(dt, 1e-3))) // 64 * 64)
    pop = orc.canonicalize(workloads.population_mix(SEED, planted, P))
    params = orc.default_params(pop=P, elite=10, p_m=2.0 / N, tol=-1.0, seed=SEED)
    for g in range(W):
        pop = oracle_generation(orc, C, pop, params, g)
    t = time.perf_counter()
    for g in range(K):
        pop = oracle_generation(orc, C, pop, params, W + g)
    dt = time.perf_counter() - t
    ms = 1000.0 * dt / max(1, K)
    value = N * N * P / (ms / 1000.0)
    cores = os.cpu_count() or 1
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "pair-updates/s",
        "n_gpus": args.gpus, "steps": K, "warmup": W, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (Noh-model returns, seed 50004)",
        "config": {"workload": "C4 (N=500; oracle on a bounded sample of P=%d chromosomes per "
                               "generation)" % P, "N": N, "population": P},
        "cpu_baseline": {"value": value, "unit": "pair-updates/s", "cores": cores, "cpu_model": cpu_model(),
                         "kind": "oracle",
                         "sample": "%d-chromosome C4 population, full generation (evaluate on %d "
                                   "threads + single-threaded operators)" % (P, cores)},
        "e2e": {"value": value, "unit": "pair-updates/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
def spawn_ranks(n):
    """`bench.py --gpus N` without a launcher: re-run this command under
    torch.distributed.run with N ranks on this node (rank 0 prints the line)."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(n),
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def cpu_model():
    try:
        for line in subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def main():
    global CONFIG, P_TOTAL
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="pga", choices=["pga", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--island-load", type=int, default=0,
                    help="diagnostic only: run ONE island of the G-GPU split (P/G chromosomes) on one GPU")
    ap.add_argument("--mode", default="islands", choices=["islands", "replicated"],
                    help="multi-GPU model: islands (population sharded, elite migration; default) or "
                         "replicated master-slave (one population, fitness sharded, L all-gathered; "
                         "SURVEY §8(f) f3)")
    ap.add_argument("--sparse-theta", type=float, default=None,
                    help="label-sparse threshold (pga_set_sparse_threshold; default: the library's automatic "
                         "choice, 0.25 with the cluster cache at N >= 64; 0 = dense sweep only)")
    ap.add_argument("--stream", action="store_true",
                    help="F1 only: each step also computes the 1760 windows on the device from one "
                         "return stream (EWMA lambda=0.98 + RMT cleaning, SURVEY §8(f) f4)")
    ap.add_argument("--fitness-only", action="store_true",
                    help="a step is one fitness evaluation of the whole population (pga_evaluate_device over "
                         "SURVEY §8(d)'s equal-thirds population mix); BASELINE configs[4] (C5) is stated "
                         "this way")
    ap.add_argument("--config", default=CONFIG, choices=sorted(CFG_POP) + ["F1"],
                    help="workload (default C4, the config the metric is quoted on; F1 = the "
                         "batched GA over 1760 windows x 18 stocks, SURVEY §8(f))")
    args = ap.parse_args()
    CONFIG = args.config
    args.warmup = max(3, args.warmup)
    ws = os.environ.get("WORLD_SIZE")
    if ws is None and args.gpus > 1:
        return spawn_ranks(args.gpus)
    if ws is not None and int(ws) != args.gpus:
        print("bench.py: WORLD_SIZE=%s but --gpus %d; launch one rank per GPU" % (ws, args.gpus),
              file=sys.stderr)
        return 2
    if CONFIG == "F1":
        return reference_f1(args) if args.impl == "reference" else bench_f1(args)
    P_TOTAL = CFG_POP[CONFIG]
    if args.impl == "reference":
        return run_reference(args)
    if args.fitness_only:
        return bench_fitness(args)

    import torch
    import torch.distributed as dist
    import paper_1403_4099_b200 as pga
    from paper_1403_4099_b200.islands import GpuIsland, IslandRunner
    from paper_1403_4099_b200.replicated import GpuReplica, ReplicatedRunner
    replicated = args.mode == "replicated"

    rank, world, local = env_int("RANK", 0), env_int("WORLD_SIZE", 1), env_int("LOCAL_RANK", 0)
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    K, W = args.steps, args.warmup

    X, planted = workloads.noh_returns(workloads.CONFIGS[CONFIG])
    N = X.shape[1]
    C = pga.pga_correlation(X, device=local)        # Eq. 7 on the device
    P_local = P_TOTAL if replicated else P_TOTAL // max(world, args.island_load)
    pm = 0.1 if N <= 40 else 2.0 / N            # Table 3 for N <= 40, else 2/N (Q13)
    params = pga.pga_params_default(
        pop_size=P_local, elite=10, p_mutation=pm, tol=-1.0, max_gens=W + K + 200,
        device=local, island=0 if replicated else rank, n_islands=1 if replicated else world,
        migrate_every=10, migrants=10, seed=SEED)

    if replicated:
        eng = GpuReplica(C, params)
        runner = ReplicatedRunner(eng)
    else:
        eng = GpuIsland(C, params)
        runner = IslandRunner(eng)
    if args.sparse_theta is not None:
        pga.pga_set_sparse_threshold(eng.ctx, args.sparse_theta)
    eng.init(SEED)
    stream = eng.stream
    for _ in range(W):
        runner.step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(list(range(torch.cuda.device_count())) if world > 1 else [local])
    if rank == 0:
        clocks.start()
        time.sleep(0.3)
    pga.pga_profile_enable(eng.ctx, True)
    launches0 = pga.pga_launch_count()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ev0.record(stream)
    for _ in range(K):
        runner.step()
    ev1.record(stream)
    torch.cuda.synchronize()
    launches = pga.pga_launch_count() - launches0
    ms = ev0.elapsed_time(ev1)
    prof = pga.pga_profile_read(eng.ctx)
    sparse_blocks, sparse_gathers = pga.pga_profile_sparse(eng.ctx)
    cache_hits, cache_saved = pga.pga_profile_cache(eng.ctx)
    pga.pga_profile_enable(eng.ctx, False)
    # roofline pass for the dense sweep kernel, right after the timed region:
    # the same population with the label-sparse pre-pass off, so every block
    # runs k_fitness (in the timed region the pre-pass may take them all)
    pga.pga_set_sparse_threshold(eng.ctx, 0.0)
    pga.pga_profile_enable(eng.ctx, 1)
    rgens = min(K, 50)
    for _ in range(rgens):
        runner.step()
    dprof = pga.pga_profile_read(eng.ctx)
    pga.pga_profile_enable(eng.ctx, False)
    pga.pga_set_sparse_threshold(eng.ctx, -1.0 if args.sparse_theta is None else args.sparse_theta)
    # diagnostic per-phase breakdown, OUTSIDE the timed region (level-2 marks)
    pga.pga_profile_enable(eng.ctx, 2)
    for _ in range(min(K, 20)):
        runner.step()
    phases, _ = pga.pga_profile_phases(eng.ctx)
    pga.pga_profile_enable(eng.ctx, False)
    # parity probe for the report (checked by the oracle in the cpu_baseline
    # leg): one more evaluation, whose labels and L are read back together
    probe = None
    if not replicated and world == 1:
        runner.e.gen_evaluate()
        probe = pga.pga_get_population(eng.ctx)
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    clk = clocks.stop() if rank == 0 else None
    st = eng.state()
    planted_L = float(pga.pga_evaluate(eng.ctx, planted[None, :].astype(np.int32) + 1)[0])

    ms_step = ms / K
    nominal = float(N) * N * P_TOTAL
    P_eval = (runner.end - runner.begin) if replicated else P_local   # chromosomes evaluated here
    executed_local = N * (N - 1) / 2.0 * P_eval
    value = nominal / (ms_step / 1000.0)

    # rooflines of the two fitness kernels from live CUDA events on the
    # library's stream (pga_profile_*), averaged over the timed generations
    ngen = max(1, prof["count"])
    sweep_ms = prof["sweep_ms"] / ngen
    sparse_ms = prof["fold_ms"] / ngen
    gen_ms = prof["gen_ms"] / ngen
    nblk = (P_eval + 31) // 32
    dense_blocks = nblk * prof["count"] - sparse_blocks
    dense_sweep_ms = dprof["sweep_ms"] / max(1, dprof["count"])       # dense roofline pass
    peaks = measured_peaks()
    sm_max = float(peaks.get("sm_max_mhz", 1965.0))
    hbm_gbs = float(peaks.get("hbm_gbs", 6542.7))
    alu_peak = ALU_PAIRS_PER_CLK * SM_COUNT * sm_max * 1e6          # SURVEY §8(d) headline ceiling
    fp64_peak = FP64_LANES_PER_SM * SM_COUNT * sm_max * 1e6
    issue_peak = 4.0 * SM_COUNT * sm_max * 1e6
    alg_bytes = P_eval * (N * 2 + 8 + 2)       # §8(d): N u16 labels read, L (f64) + top (u16) written
    tj = {}
    if world == 1:
        try:
            tj = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
        except Exception:
            tj = {}
    cfg_key = "%s_w%d" % (CONFIG, 1)
    sp_ncu = tj.get("k_fitness_sparse", {}).get(cfg_key, {})
    dn_ncu = tj.get("k_fitness", {}).get(cfg_key, {})

    achieved = executed_local / (dense_sweep_ms / 1000.0)
    rl_dense = {
        "bound": "alu", "kernel": "k_fitness (TMA pair sweep + fused fold)",
        "achieved": achieved, "peak": alu_peak, "unit": "pair-updates/s", "frac": achieved / alu_peak,
        "traffic": dn_ncu.get("dram_bytes_per_launch"), "algorithmic_bytes": alg_bytes,
        "work_per_launch": "%d chromosomes x N(N-1)/2 = %.4g executed pair-updates" % (P_eval, executed_local),
        "peak_basis": "SURVEY §8(d): ISETP+SEL per pair on the 64-op/clk/SM INT pipe = 32 pairs/clk/SM "
                      "x 148 SMs x %.0f MHz (sm_max_mhz)" % sm_max,
        "measured": "CUDA events on the library stream over %d generations right after the timed region "
                    "(same population, label-sparse pass off, so every block runs k_fitness): %.4f ms "
                    "per launch.  In the timed region k_fitness ran %.1f%% of the blocks (%.4f ms per "
                    "generation)" % (dprof["count"], dense_sweep_ms, 100.0 * dense_blocks / float(nblk * ngen),
                                     sweep_ms),
        "other_bounds": [
            {"bound": "fp64", "peak": fp64_peak, "frac": achieved / fp64_peak,
             "basis": "1 DADD per executed pair, 64 FP64 lanes/clk/SM"},
            {"bound": "measured_loop", "peak": LOOP_PAIRS_PER_CLK * SM_COUNT * sm_max * 1e6,
             "frac": achieved / (LOOP_PAIRS_PER_CLK * SM_COUNT * sm_max * 1e6),
             "basis": "tools/mb_pairloop.cu bare inner loop: 26.8 pairs/clk/SM"},
            {"bound": "hbm", "achieved_gbs": alg_bytes / (dense_sweep_ms / 1000.0) / 1e9, "peak_gbs": hbm_gbs,
             "frac": alg_bytes / (dense_sweep_ms / 1000.0) / 1e9 / hbm_gbs},
        ],
    }
    rl_sparse = None
    if prof["fold_ms"] > 0 and sparse_blocks > 0:
        sp_s = sparse_ms / 1000.0
        pairs_needed = (sparse_gathers + cache_saved) / float(ngen)   # sum n_s(n_s-1)/2 per launch
        gbs = alg_bytes / sp_s / 1e9
        others = [
            {"bound": "alu", "what": "necessary pair-updates per launch (C entries gathered + pair updates "
                                     "served by the cluster cache) = %.4g" % pairs_needed,
             "achieved": pairs_needed / sp_s, "peak": alu_peak, "unit": "pair-updates/s",
             "frac": pairs_needed / sp_s / alu_peak},
            {"bound": "l2_gather", "what": "C entries gathered from L2 per launch = %.4g"
                                           % (sparse_gathers / float(ngen)),
             "achieved": sparse_gathers / float(ngen) / sp_s, "peak": L2_GATHERS_PER_S, "unit": "gathers/s",
             "frac": sparse_gathers / float(ngen) / sp_s / L2_GATHERS_PER_S,
             "basis": "tools/mb_l2gather.cu: 3.03e11 random 8-byte gathers/s from an L2-resident C"},
        ]
        if sp_ncu.get("inst_per_launch"):
            others.append({"bound": "issue", "what": "%.4g warp-instructions per launch (ncu "
                                                      "smsp__inst_executed.sum, %s)" % (sp_ncu["inst_per_launch"],
                                                                                        sp_ncu.get("source", "")),
                           "achieved": sp_ncu["inst_per_launch"] / sp_s, "peak": issue_peak,
                           "unit": "warp-instructions/s", "frac": sp_ncu["inst_per_launch"] / sp_s / issue_peak,
                           "basis": "1 warp-instruction/clk per SMSP, 4 per SM"})
        rl_sparse = {
            "bound": "hbm", "kernel": "k_fitness_sparse (label-sparse pass + cluster cache)",
            "achieved": gbs, "peak": hbm_gbs, "unit": "GB/s", "frac": gbs / hbm_gbs,
            "traffic": sp_ncu.get("dram_bytes_per_launch"), "algorithmic_bytes": alg_bytes,
            "work_per_launch": "%d chromosomes x (2N label bytes + 8 B L + 2 B top) = %d algorithmic bytes"
                               % (P_eval, alg_bytes),
            "measured": "CUDA events on the library stream around every k_fitness_sparse launch of the timed "
                        "region: %.4f ms per launch of %.4f ms per generation" % (sparse_ms, gen_ms),
            "traffic_note": "ncu dram__bytes_read+write of one launch inside the bench window (%s)"
                            % sp_ncu.get("source", "no capture for this config"),
            "other_bounds": others,
            "cluster_cache": {"hits_per_launch": cache_hits / float(ngen),
                              "pair_updates_saved_per_launch": cache_saved / float(ngen),
                              "hit_share_of_pairs": cache_saved / float(max(1, cache_saved + sparse_gathers))},
            "share_of_timed_generation": sparse_ms / gen_ms,
        }

    # end-to-end through the public API from host memory (rank-local), see DESIGN.md §7
    e2e = None
    if not args.no_e2e and not replicated:
        eng.close()
        e2e = e2e_run(pga, torch, dist, C, params, world, K, planted, args.sparse_theta)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        v, Ps, ng, dt, v1 = oracle_rate(C, planted, max_P=P_TOTAL)
        cores = os.cpu_count() or 1
        cpu = {"value": v, "unit": "pair-updates/s", "cores": cores, "cpu_model": cpu_model(),
               "kind": "oracle",
               "sample": "%d-chromosome %s population, %d full oracle generations (evaluate on "
                         "%d host threads + single-threaded operators), %.1f s"
                         % (Ps, CONFIG, ng, cores, dt),
               "single_thread_evaluate": {"value": v1, "unit": "pair-updates/s", "cores": 1}}
        if probe is not None:
            cpu["parity"] = parity_probe(C, probe[0] - 1, probe[1], cores)
    if eng.ctx is not None:
        eng.close()

    if rank == 0:
        # the top-level roofline is the kernel that dominated the timed region
        if rl_sparse is not None and sparse_ms > sweep_ms:
            rl_main, rl_other = rl_sparse, rl_dense
        else:
            rl_main, rl_other = rl_dense, rl_sparse
        line = {
            "metric": METRIC, "value": value, "unit": "pair-updates/s", "n_gpus": world,
            "steps": K, "warmup": W, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (Noh-model returns T=%d, seed %d; Pearson C on device)"
                    % (workloads.CONFIGS[CONFIG].T, workloads.CONFIGS[CONFIG].seed),
            "config": {"workload": "%s: N=%d, P=%d total (%d per GPU), 1 step = 1 generation"
                                   % (CONFIG, N, P_TOTAL, P_local), "N": N, "population": P_TOTAL,
                       "population_per_gpu": P_local,
                       **({"diagnostic_island_load_of_gpus": args.island_load} if args.island_load else {}),
                       "parallelism": ("replicated master-slave x%d (fitness shard %d per GPU)"
                                       % (world, P_eval)) if replicated else "islands x%d" % world,
                       "migration": "none: L and top all-gathered every generation (NCCL)"
                                    if replicated else "every 10 generations, 10 elites, NCCL all-gather",
                       "l2": ("working set > L2 (two population layouts x2 buffers + 264 MB "
                              "fold scratch per GPU); no flush") if N * P_local >= 8000000 else
                             "working set fits L2 (small config; timing is launch/latency-bound)"},
            "evals_per_s": P_TOTAL / (ms_step / 1000.0),
            "gens_per_s": 1000.0 / ms_step,
            "dense_equivalent_pair_updates_per_s": executed_local * world / (ms_step / 1000.0),
            "kernel_ms_per_generation": {"k_fitness": sweep_ms, "k_fitness_sparse": sparse_ms,
                                         "generation": gen_ms,
                                         "k_fitness_dense_pass": dense_sweep_ms},
            "sparse_pass": {"blocks_evaluated_sparsely": sparse_blocks,
                            "fraction_of_blocks": sparse_blocks / float(nblk * ngen),
                            "note": "SURVEY §8(f) f2: blocks of 32 chromosomes whose clusters need <= 25% "
                                    "of the dense pair updates (automatic threshold with the cluster "
                                    "cache on) are evaluated label-sparsely and skipped by k_fitness; "
                                    "clusters of >= 4 genes come from the cluster cache when an earlier "
                                    "generation had the same member set, the rest are gathered from L2"},
            "phase_ms_per_generation": {("stats_order_selection" if k == "stats" else k): round(v, 4)
                                        for k, v in phases.items() if k != "fitness_fold_fused"},
            "phase_note": "diagnostic pass after the timed region (phase events add ~3 us/gen); in "
                          "non-migration generations the order sort and the selection run in phase A "
                          "beside the statistics (side stream), so their time is in "
                          "stats_order_selection and order_sort/selection/mates show only the marks",
            "roofline": rl_main,
            "roofline_other": rl_other,
            "gpu_launches": int(launches),
            "clocks": clk,
            "best_L": st["best_L"],
            "planted": {"L": planted_L, "best_L_reached": st["best_L"],
                        "note": "planted partition's Eq. 8 value (pga_evaluate) vs the GA's best after the "
                                "timed window; C4 reaches the planted partition exactly by ~5000 generations "
                                "(tests/test_gpu_parity.py::test_run_recovers_planted_C4)"},
            "e2e": e2e,
            "cpu_baseline": cpu,
            "parity": (cpu or {}).get("parity"),
            "paper_context": "Table 4 (P:369, P:373): the paper's CUDA PGA clusters one 18-stock JSE "
                             "correlation matrix in 0.80 s median on a GTX Titan Black (1.39 s on a Tesla "
                             "C2050; serial MATLAB 7.77 s), population 1000, <= 400 generations; at most "
                             "~5e5 fitness evaluations/s (BASELINE.md §1).  Other hardware, data and "
                             "workload: context, not a target.",
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def bench_fitness(args):
    """Fitness-only throughput (BASELINE configs[4]: C5, N = 2000, P = 262144,
    "fitness-eval-only throughput sweep"): a step is one pga_evaluate_device
    over the whole population, the equal-thirds mix of SURVEY §8(d) (8192
    base rows repeated under per-copy label permutations, built on the
    device).  Weak scaling over ranks (each rank evaluates its own P)."""
    import torch
    import torch.distributed as dist
    import paper_1403_4099_b200 as pga
    rank, world, local = env_int("RANK", 0), env_int("WORLD_SIZE", 1), env_int("LOCAL_RANK", 0)
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    K, W = args.steps, args.warmup
    X, planted = workloads.noh_returns(workloads.CONFIGS[CONFIG])
    N = X.shape[1]
    C = pga.pga_correlation(X, device=local)
    P = P_TOTAL
    base_P = min(P, 8192)
    reps = (P + base_P - 1) // base_P
    base = workloads.population_mix(SEED + rank, planted, base_P)
    rng = np.random.default_rng(SEED + rank)
    perms = np.stack([rng.permutation(N) for _ in range(reps)]).astype(np.int64)
    ctx = pga.pga_create(C, pga.pga_params_default(pop_size=P, device=local))
    db = torch.from_numpy(base.astype(np.int64)).cuda()
    dp = torch.from_numpy(perms).cuda()
    dl = torch.empty((P, N), dtype=torch.int16, device="cuda")
    for t in range(reps):
        n = min(base_P, P - t * base_P)
        dl[t * base_P:t * base_P + n] = torch.gather(dp[t].expand(base_P, N), 1, db)[:n].to(torch.int16)
    del db
    # re-evaluating one population would let the cluster cache serve every
    # large cluster from the previous step (memoised outputs): off here
    pga.pga_set_cluster_cache(ctx, 0)
    if args.sparse_theta is not None:
        pga.pga_set_sparse_threshold(ctx, args.sparse_theta)
    L = torch.zeros(P, dtype=torch.float64, device="cuda")
    stream = torch.cuda.current_stream()
    for _ in range(W):
        pga.pga_evaluate_device(ctx, dl, L, stream=stream.cuda_stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(list(range(torch.cuda.device_count())) if world > 1 else [local])
    if rank == 0:
        clocks.start()
        time.sleep(0.3)
    b0, g0 = pga.pga_profile_sparse(ctx)
    launches0 = pga.pga_launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    ev0.record(stream)
    for _ in range(K):
        pga.pga_evaluate_device(ctx, dl, L, stream=stream.cuda_stream)
    ev1.record(stream)
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    launches = pga.pga_launch_count() - launches0
    b1, g1 = pga.pga_profile_sparse(ctx)
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    clk = clocks.stop() if rank == 0 else None
    Lg = L.cpu().numpy()
    ms_step = ms / K
    nblk = (P + 31) // 32
    sparse_frac = (b1 - b0) / float(nblk * K)
    executed = N * (N - 1) / 2.0 * P
    peaks = measured_peaks()
    sm_max = float(peaks.get("sm_max_mhz", 1965.0))
    alu_peak = ALU_PAIRS_PER_CLK * SM_COUNT * sm_max * 1e6
    hbm = float(peaks.get("hbm_gbs", 6542.7))
    alg_bytes = P * (N * 2 + 8)
    dense_rate = executed * (1.0 - sparse_frac) / (ms_step / 1000.0)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        import oracle as orc
        orc.build()
        Ch = orc.pearson(X)
        idx = np.unique(np.concatenate([rng.choice(P, 1024, replace=False), [0, P - 1]]))
        rows = np.stack([perms[i // base_P][base[i % base_P]] for i in idx]).astype(np.int32)
        cores = os.cpu_count() or 1
        t0 = time.perf_counter()
        Lo, _ = orc.evaluate(Ch, rows, nthreads=cores)
        dt = time.perf_counter() - t0
        err = np.abs(Lg[idx] - Lo) / np.maximum(1.0, np.abs(Lo))
        cpu = {"value": N * N * len(idx) / dt, "unit": "pair-updates/s", "cores": cores, "cpu_model": cpu_model(),
               "kind": "oracle", "sample": "orc_evaluate of %d sampled rows of the same population on %d host "
                                          "threads, %.1f s" % (len(idx), cores, dt),
               "parity": {"rows": int(len(idx)), "max_rel_dL": float(err.max()), "tolerance": 1e-9,
                          "pass": bool(err.max() <= 1e-9)}}
    pga.pga_destroy(ctx)
    if rank == 0:
        line = {
            "metric": "fitness evaluation throughput, nominal pair-updates/s (N^2 * P per evaluation)",
            "value": float(N) * N * P * world / (ms_step / 1000.0), "unit": "pair-updates/s", "n_gpus": world,
            "steps": K, "warmup": W, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (Noh-model returns, seed %d; Pearson C on device; equal-thirds label mix)"
                    % workloads.CONFIGS[CONFIG].seed,
            "config": {"workload": "%s fitness only: N=%d, P=%d per GPU, 1 step = 1 evaluation of the population"
                                   % (CONFIG, N, P), "N": N, "population_per_gpu": P,
                       "l2": "working set > L2 (labels %.0f MB per GPU); no flush" % (P * N * 2 / 1e6)},
            "evals_per_s": P * world / (ms_step / 1000.0),
            "sparse_block_fraction": sparse_frac,
            "cluster_cache": "off (the same population is evaluated every step; cached terms would be memoised "
                             "outputs)",
            "roofline": {"bound": "alu", "kernel": "k_fitness (dense sweep; the label-sparse pass took %.1f%% "
                                                   "of the blocks)" % (100 * sparse_frac),
                         "achieved": dense_rate, "peak": alu_peak, "unit": "pair-updates/s",
                         "frac": dense_rate / alu_peak,
                         "traffic": None, "algorithmic_bytes": alg_bytes,
                         "work_per_launch": "dense blocks x 32 chromosomes x N(N-1)/2 executed pair-updates",
                         "peak_basis": "SURVEY §8(d): 32 pairs/clk/SM x 148 x %.0f MHz" % sm_max,
                         "other_bounds": [{"bound": "hbm", "achieved_gbs": alg_bytes / (ms_step / 1000.0) / 1e9,
                                           "peak_gbs": hbm,
                                           "frac": alg_bytes / (ms_step / 1000.0) / 1e9 / hbm}],
                         "measured": "CUDA events around K evaluate launches on the caller stream"},
            "gpu_launches": int(launches), "clocks": clk, "cpu_baseline": cpu,
            "parity": (cpu or {}).get("parity"),
            "e2e": None,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def reference_f1(args):
    """--impl reference for F1: orc_run per window on the host, each step a
    bounded sample of windows (single-threaded)."""
    if env_int("RANK", 0) != 0:
        return 0
    import oracle as orc
    orc.build()
    f1 = workloads.F1
    K, W = args.steps, args.warmup
    budget = 150.0 / max(1, K + W)
    X, _ = workloads.window_returns(64, f1["N"], f1["T"], f1["seed0"])
    Cs = [orc.pearson(X[b]) for b in range(64)]
    op = orc.default_params(pop=f1["pop"], max_gens=f1["gens"])
    done, t_all = 0, 0.0
    for s in range(W + K):
        t0 = time.perf_counter()
        n = 0
        while n == 0 or time.perf_counter() - t0 < budget:
            op.seed = SEED + (done % 64)
            orc.run(Cs[done % 64], op, nthreads=1)
            done += 1
            n += 1
        if s >= W:
            t_all += time.perf_counter() - t0
            nk = n
    value = nk / (t_all / K) if K else 0.0
    line = {"impl": "reference", "metric": "batched GA: correlation matrices clustered per second "
            "(each window its own Table 3 GA run to termination)", "value": value,
            "unit": "matrices/s", "n_gpus": args.gpus, "steps": K, "warmup": W,
            "ms_per_step": 1000.0 * t_all / max(1, K), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (F1 windows)",
            "config": {"workload": "F1 windows, oracle orc_run single-threaded"},
            "cpu_baseline": {"value": value, "unit": "matrices/s", "cores": 1, "kind": "oracle",
                             "sample": "windows run to termination within each ~%.0f s step" % budget},
            "e2e": {"value": value, "unit": "matrices/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def bench_f1(args):
    """F1: the batched GA.  One step = one complete
    pga_batch_run over B = 1760 windows of N = 18 stocks (each window its own
    GA, Table 3 configuration, stall termination), the paper's test-set
    shape (Table 4 P:356-375 times it at 0.80 s per matrix on a GTX
    Titan Black).  Windows shard over ranks (weak scaling: 1760 per GPU)."""
    import torch
    import torch.distributed as dist
    import paper_1403_4099_b200 as pga
    rank, world, local = env_int("RANK", 0), env_int("WORLD_SIZE", 1), env_int("LOCAL_RANK", 0)
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    K, W = args.steps, args.warmup
    f1 = workloads.F1
    B, N, T = f1["B"], f1["N"], f1["T"]
    stride = 10
    if args.stream:
        # one return stream; window b = EWMA state after observation T-1 + b*stride, RMT-cleaned
        Ts = T + (B - 1) * stride
        Xs, planted1 = workloads.stream_returns(Ts, N, seed=f1["seed0"] + rank)
        planted = np.tile(planted1, (B, 1))
        dXs = torch.from_numpy(Xs).cuda()
        dC = torch.empty((B, N, N), dtype=torch.float64, device="cuda")
        status = torch.zeros(1, dtype=torch.int32, device="cuda")
        pga.pga_corr_stream_device(dXs, dC, status, lam=0.98, warm=T, stride=stride, q=0.0,
                                   device=local, stream=torch.cuda.current_stream().cuda_stream)
        assert int(status.item()) == 0
    else:
        X, planted = workloads.window_returns(B, N, T, f1["seed0"] + rank * B)
        dX = torch.from_numpy(X).cuda()
        dC = torch.empty((B, N, N), dtype=torch.float64, device="cuda")
        status = torch.zeros(B, dtype=torch.int32, device="cuda")
        for b in range(B):                              # Eq. 7 on the device
            pga.pga_correlation_device(dX[b], dC[b], status[b:b + 1])
        torch.cuda.synchronize()
        assert int(status.sum()) == 0
    params = pga.pga_params_default(pop_size=f1["pop"], max_gens=f1["gens"], seed=SEED + rank * B,
                                    device=local)
    lab = torch.zeros((B, N), dtype=torch.int32, device="cuda")
    bL = torch.zeros(B, dtype=torch.float64, device="cuda")
    gens = torch.zeros(B, dtype=torch.int32, device="cuda")
    reason = torch.zeros(B, dtype=torch.int32, device="cuda")
    stream = torch.cuda.current_stream()

    def step():
        if args.stream:
            pga.pga_corr_stream_device(dXs, dC, status, lam=0.98, warm=T, stride=stride, q=0.0,
                                       device=local, stream=stream.cuda_stream)
        pga.pga_batch_run_device(dC, params, lab, bL, gens, reason, stream=stream.cuda_stream)

    for _ in range(W):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(list(range(torch.cuda.device_count())) if world > 1 else [local])
    if rank == 0:
        clocks.start()
        time.sleep(0.3)
    launches0 = pga.pga_launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ev0.record(stream)
    for _ in range(K):
        step()
    ev1.record(stream)
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    launches = pga.pga_launch_count() - launches0
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    clk = clocks.stop() if rank == 0 else None
    ms_step = ms / K
    g = gens.cpu().numpy().astype(np.int64)
    evals = int(g.sum()) * f1["pop"]
    executed = evals * N * (N - 1) / 2.0
    value = B * world / (ms_step / 1000.0)
    peaks = measured_peaks()
    sm_max = float(peaks.get("sm_max_mhz", 1965.0))
    peak = FP64_LANES_PER_SM * SM_COUNT * sm_max * 1e6
    achieved = executed / (ms_step / 1000.0)
    best = lab.cpu().numpy() - 1
    same = float(np.mean([np.array_equal(best[b], planted[b]) for b in range(B)]))
    f1_traffic = f1_inst = None
    try:
        tj = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
        f1_traffic = tj.get("k_batch", {}).get("dram_bytes_per_launch")
        f1_inst = tj.get("k_batch", {}).get("inst_per_launch")
    except Exception:
        pass

    # e2e: the host-memory call (C from pinned host, results back to host)
    e2e = None
    if not args.no_e2e:
        Cp = torch.from_numpy(dC.cpu().numpy()).pin_memory()
        if args.stream:
            Xp = torch.from_numpy(Xs).pin_memory()
        ke = max(1, min(K, 3))
        # one untimed call first: the host path's first call also creates the
        # stream-ordered memory pool (~80 ms once per process)
        if args.stream:
            pga.pga_batch_run(pga.pga_corr_stream(Xp.numpy(), lam=0.98, warm=T, stride=stride, q=0.0,
                                                  device=local), params)
        else:
            pga.pga_batch_run(Cp.numpy(), params)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(ke):
            Cin = pga.pga_corr_stream(Xp.numpy(), lam=0.98, warm=T, stride=stride, q=0.0,
                                      device=local) if args.stream else Cp.numpy()
            res = pga.pga_batch_run(Cin, params)
        dt = (time.perf_counter() - t0) / ke
        if world > 1:
            t = torch.tensor([dt], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = float(t.item())
        h2d = (Xs.size * 8 + B * N * N * 8) if args.stream else B * N * N * 8
        e2e = {"value": B * world / dt, "unit": "matrices/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": B * (N * 4 + 8 + 4 + 4) + (B * N * N * 8 if args.stream else 0),
               "steps": ke, "seconds_per_step": dt,
               "includes": ("pga_corr_stream with host returns (upload, EWMA/RMT, download) + "
                            if args.stream else "") +
                           "pga_batch_run with host buffers: C upload, run, results download"}
        assert np.array_equal(res["best_labels"], lab.cpu().numpy())

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        import oracle as orc
        orc.build()
        Ch = dC.cpu().numpy()
        op = orc.default_params(pop=f1["pop"], max_gens=f1["gens"])
        t0 = time.perf_counter()
        nb = 0
        while nb < B and time.perf_counter() - t0 < 15.0:
            op.seed = SEED + nb
            orc.run(Ch[nb], op, nthreads=1)
            nb += 1
        dt = time.perf_counter() - t0
        cpu = {"value": nb / dt, "unit": "matrices/s", "cores": 1, "kind": "oracle",
               "sample": "orc_run on the first %d windows (single-threaded), %.1f s" % (nb, dt)}

    if rank == 0:
        line = {
            "metric": "batched GA: correlation matrices clustered per second "
                      "(each window its own Table 3 GA run to termination)",
            "value": value, "unit": "matrices/s", "n_gpus": world, "steps": K, "warmup": W,
            "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64",
            "data": ("synthetic (one Noh-model return stream of %d observations, seed %d; windows = "
                     "EWMA/RMT states every %d observations, computed on device)"
                     % (T + (B - 1) * stride, f1["seed0"] + rank, stride)) if args.stream else
                    "synthetic (Noh-model windows, T=160, seeds %d+b; Pearson C on device)" % f1["seed0"],
            "config": {"workload": "F1%s: B=%d windows per GPU x N=%d stocks, population %d, <= %d "
                                   "generations, stall 50 / tol 1e-5; 1 step = all windows"
                                   % (" + stream (returns -> EWMA/RMT windows on device)" if args.stream
                                      else "", B, N, f1["pop"], f1["gens"]),
                       "B_per_gpu": B, "N": N, "population": f1["pop"],
                       "parallelism": "windows sharded x%d" % world,
                       "l2": "C (4.6 MB) read once per step; state lives in shared memory"},
            "paper_context": "Table 4 (P:369): 0.80 s per matrix = 1.25 matrices/s on a GTX Titan "
                             "Black (JSE data, not this synthetic set)",
            "generations_mean": float(g.mean()), "generations_max": int(g.max()),
            "evals_per_s": evals * world / (ms_step / 1000.0),
            "planted_equals_best": same,
            "roofline": ({"bound": "issue", "kernel": "k_batch",
                          "achieved": f1_inst / (ms_step / 1000.0),
                          "peak": 4.0 * SM_COUNT * sm_max * 1e6, "unit": "warp-instructions/s",
                          "frac": f1_inst / (ms_step / 1000.0) / (4.0 * SM_COUNT * sm_max * 1e6),
                          "traffic": f1_traffic, "algorithmic_bytes": B * N * N * 8 + B * (N * 4 + 16),
                          "work_per_launch": "%.4g warp-instructions (ncu smsp__inst_executed.sum of one "
                                             "launch, profiles/traffic.json) / the step time" % f1_inst,
                          "peak_basis": "4 warp-instructions/clk/SM x 148 SMs x %.0f MHz: at N=18 the "
                                        "GA operators (sort, selection, Philox, breed) are most of the "
                                        "kernel, so instruction issue, not the FP64 pipe, bounds it"
                                        % sm_max}
                         if f1_inst else None),
            "roofline_other": {"bound": "alu", "kernel": "k_batch", "achieved": achieved, "peak": peak,
                               "unit": "pair-updates/s", "frac": achieved / peak,
                               "work_per_launch": "sum over windows of gens x %d chromosomes x N(N-1)/2"
                                                  % f1["pop"],
                               "note": "the fitness pairs alone against the FP64 bound"},
            "gpu_launches": int(launches), "clocks": clk, "e2e": e2e, "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def e2e_run(pga, torch, dist, C, params, world, K, planted, theta=None):
    """Same metric through the public API with HOST buffers: C copied from
    pinned host memory (pga_create), K generations, and every step a
    device->host read of the step's result (best L, mean L, best labels)."""
    from paper_1403_4099_b200.islands import GpuIsland, IslandRunner
    N = C.shape[0]
    Cp = torch.from_numpy(np.ascontiguousarray(C)).pin_memory()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    eng = GpuIsland(Cp.numpy(), params)
    runner = IslandRunner(eng)
    if theta is not None:
        pga.pga_set_sparse_threshold(eng.ctx, theta)
    eng.init(SEED)
    for _ in range(K):
        runner.step()
        st = eng.state()                 # D2H of the step's result (syncs)
    bestL, best, _ = runner.global_best()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([dt], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dt = float(t.item())
    eng.close()
    value = float(N) * N * P_TOTAL * K / dt
    d2h = 56 + 2 * N          # DevState + best labels (u16)
    return {"value": value, "unit": "pair-updates/s", "h2d_bytes_per_step": N * N * 8 / K,
            "d2h_bytes_per_step": d2h, "steps": K, "seconds": dt,
            "includes": "pga_create from pinned host C (device buffers from the library's memory "
                        "pool, which keeps the pages of the timed run's destroyed context) + init + K "
                        "generations + per-step state read + final global best gather"}


if __name__ == "__main__":
    sys.exit(main())
