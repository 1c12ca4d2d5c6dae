"""Replicated master-slave driver over torch.distributed (SURVEY §8(f) row
f3; the paper's parallel model, §3.2: one population, fitness
evaluated in parallel, the GA operators on the master).

Every rank holds a replica of the SAME population (n_islands = 1, same
seed).  Per generation rank r evaluates its contiguous shard
[r*S, min(P, (r+1)*S)) with S = 32 * ceil(P / (32 * world)); the ranks
all-gather L and the KB top labels (10 bytes per chromosome; NCCL over
NVLink on GPUs, gloo in CPU tests); every rank installs the full vectors and
runs the same deterministic operators, so the replicas stay bit-identical.
With the label-sparse pass off (pga_set_sparse_threshold(ctx, 0)) the run
also equals the single-GPU pga_run bit for bit; with it on, a block's path
(and so the last bits of its L) can depend on the launch history.

The driver only moves bytes and sequences calls.  ``GpuReplica`` is the
product engine; tests plug in an oracle-backed engine with the same methods.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from . import binding as B


class GpuReplica:
    """One replica = one pga_ctx (n_islands = 1) on this process's GPU."""

    def __init__(self, C, params: B.pga_params):
        if params.n_islands != 1:
            raise ValueError("replicated mode runs one population: n_islands must be 1")
        self.params = params
        self.N = int(np.asarray(C).shape[0])
        self.P = int(params.pop_size)
        self.ctx = B.pga_create(C, params)
        self.device = torch.device("cuda", params.device)
        self.stream = torch.cuda.ExternalStream(B.pga_get_stream(self.ctx), device=self.device)

    def close(self):
        if self.ctx is not None:
            B.pga_destroy(self.ctx)
            self.ctx = None

    def init(self, seed):
        B.pga_init(self.ctx, seed)

    def rep_evaluate(self, begin, end, L_out, top_out):
        B.pga_rep_evaluate(self.ctx, begin, end, L_out, top_out)

    def rep_commit(self, L, top):
        B.pga_rep_commit(self.ctx, L, top)

    def gen_breed(self):
        B.pga_gen_breed(self.ctx)

    def state(self):
        return B.pga_get_state(self.ctx, self.N)


def shard(P: int, world: int, rank: int):
    """(begin, end, S): this rank's chromosomes and the common shard size."""
    S = 32 * ((P + 32 * world - 1) // (32 * world))
    begin = min(P, rank * S)
    return begin, min(P, begin + S), S


class ReplicatedRunner:
    def __init__(self, engine, group=None):
        self.e = engine
        self.group = group
        init = dist.is_initialized()
        self.world = dist.get_world_size(group) if init else 1
        self.rank = dist.get_rank(group) if init else 0
        self.begin, self.end, self.S = shard(engine.P, self.world, self.rank)
        dev = getattr(engine, "device", torch.device("cpu"))
        self.L_send = torch.zeros(self.S, dtype=torch.float64, device=dev)
        self.t_send = torch.zeros(self.S, dtype=torch.int16, device=dev)
        self.L_recv = torch.zeros(self.S * self.world, dtype=torch.float64, device=dev)
        self.t_recv = torch.zeros(self.S * self.world, dtype=torch.int16, device=dev)

    def _allgather(self):
        if self.world == 1:
            self.L_recv.copy_(self.L_send)
            self.t_recv.copy_(self.t_send)
            return
        # 16-bit top labels travel as bytes (no int16 collectives in NCCL/gloo)
        pairs = ((self.L_send, self.L_recv),
                 (self.t_send.view(torch.uint8), self.t_recv.view(torch.uint8)))
        if dist.get_backend(self.group) == "nccl":
            for send, recv in pairs:
                dist.all_gather_into_tensor(recv, send, group=self.group)
        else:
            for send, recv in pairs:
                parts = list(recv.chunk(self.world))
                dist.all_gather(parts, send, group=self.group)
                recv.copy_(torch.cat(parts))

    def _step(self):
        n = self.end - self.begin
        if n > 0:
            self.e.rep_evaluate(self.begin, self.end, self.L_send[:n], self.t_send[:n])
        self._allgather()
        P = self.e.P
        self.e.rep_commit(self.L_recv[:P], self.t_recv[:P])
        self.e.gen_breed()

    def step(self):
        stream = getattr(self.e, "stream", None)
        if stream is not None:
            with torch.cuda.stream(stream):
                self._step()
        else:
            self._step()

    def run(self, gens):
        for _ in range(gens):
            self.step()
