"""Island-model driver over torch.distributed (P:147 ZLL2012, P:360, P:441;
reading Q21): one process per GPU, each evolving its shard of the population
as an island; every `migrate_every` generations the islands all-gather their
elite records (NCCL over NVLink on GPUs, gloo in CPU tests) and each replaces
its worst individuals with the global best (done inside the engine).

The driver only moves bytes and sequences calls; the GA arithmetic is in the
engine (libpga.so on a GPU).  ``GpuIsland`` is the product engine; tests plug
in an oracle-backed engine with the same five methods to check the exchange
logic on CPU with world_size 2.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from . import binding as B


class GpuIsland:
    """One island = one pga_ctx on this process's GPU."""

    def __init__(self, C, params: B.pga_params):
        self.params = params
        self.N = int(np.asarray(C).shape[0])
        self.ctx = B.pga_create(C, params)
        self.device = torch.device("cuda", params.device)
        self.stream = torch.cuda.ExternalStream(B.pga_get_stream(self.ctx), device=self.device)

    def close(self):
        if self.ctx is not None:
            B.pga_destroy(self.ctx)
            self.ctx = None

    # -- engine interface -------------------------------------------------
    def init(self, seed):
        B.pga_init(self.ctx, seed)

    def gen_evaluate(self) -> bool:
        return B.pga_gen_evaluate(self.ctx)

    def gen_breed(self):
        B.pga_gen_breed(self.ctx)

    def migrant_bytes(self) -> int:
        return B.pga_migrant_bytes(self.ctx)

    def export_migrants(self, send: torch.Tensor):
        B.pga_export_migrants(self.ctx, send)

    def import_migrants(self, recv: torch.Tensor, n_islands: int):
        B.pga_import_migrants(self.ctx, recv, n_islands)

    def state(self):
        return B.pga_get_state(self.ctx, self.N)


class IslandRunner:
    """Drives one island and its exchanges.  `group` may be None (single
    island: the all-gather degenerates to a copy)."""

    def __init__(self, engine, group=None):
        self.e = engine
        self.group = group
        self.world = dist.get_world_size(group) if group is not None or dist.is_initialized() else 1
        nb = engine.migrant_bytes()
        dev = getattr(engine, "device", torch.device("cpu"))
        self.send = torch.zeros(nb, dtype=torch.uint8, device=dev)
        self.recv = torch.zeros(nb * self.world, dtype=torch.uint8, device=dev)
        self.exchanges = 0

    def _allgather(self):
        if self.world == 1:
            self.recv.copy_(self.send)
        elif dist.get_backend(self.group) == "nccl":
            dist.all_gather_into_tensor(self.recv, self.send, group=self.group)
        else:  # gloo (CPU tests): list form
            parts = list(self.recv.chunk(self.world))
            dist.all_gather(parts, self.send, group=self.group)
            self.recv.copy_(torch.cat(parts))
        self.exchanges += 1

    def step(self):
        """One generation: phase A, [migration], phase B."""
        mig = self.e.gen_evaluate()
        if mig:
            stream = getattr(self.e, "stream", None)
            if stream is not None:
                with torch.cuda.stream(stream):
                    self.e.export_migrants(self.send)
                    self._allgather()
                    self.e.import_migrants(self.recv, self.world)
            else:
                self.e.export_migrants(self.send)
                self._allgather()
                self.e.import_migrants(self.recv, self.world)
        self.e.gen_breed()
        return mig

    def run(self, gens):
        """Up to `gens` generations; stops once the engine reports termination
        (Q28: every island decides identically, so all ranks stop together).
        Returns the generations stepped."""
        for g in range(gens):
            self.step()
            if self.e.state().get("done"):
                return g + 1
        return gens

    def global_best(self):
        """(best L, labels) over all islands: (L desc, island asc)."""
        st = self.e.state()
        N = len(st["best_labels"])
        rec = torch.zeros(1 + N, dtype=torch.float64)
        rec[0] = st["best_L"]
        rec[1:] = torch.from_numpy(st["best_labels"].astype(np.float64))
        if self.world > 1:
            dev = getattr(self.e, "device", torch.device("cpu"))
            r = rec.to(dev)
            parts = [torch.zeros_like(r) for _ in range(self.world)]
            dist.all_gather(parts, r, group=self.group)
            allr = torch.stack(parts).cpu()
        else:
            allr = rec.view(1, 1 + N)
        k = int(torch.argmax(allr[:, 0]).item())   # first max = lowest island
        return float(allr[k, 0]), allr[k, 1:].numpy().astype(np.int32), k
