"""An oracle-backed island engine (TEST INFRASTRUCTURE) with the same
interface as paper_1403_4099_b200.islands.GpuIsland, so the island driver and
its collectives can be exercised on CPU (gloo, world_size 2).  The record
layout it exports/imports is the one libpga.so uses (include/pga.h:
{f64 L, u16 top, pad, u16 labels[N]} padded to 16 bytes)."""
import numpy as np
import torch

import oracle as orc


class OracleIsland:
    def __init__(self, C, params, island, n_islands):
        self.C = np.ascontiguousarray(C, np.float64)
        self.N = self.C.shape[0]
        self.p = params
        self.island = island
        self.G = n_islands
        self.P = params.pop
        self.rec = (16 + 2 * self.N + 15) // 16 * 16
        self.device = torch.device("cpu")

    def init(self, seed):
        self.p.seed = seed
        self.pop = orc.init_population(seed, self.N, self.P, p_off=self.island * self.P,
                                       island=self.island)
        self.gen = 0
        self.best_ever = -1.0
        self.best_labels = np.zeros(self.N, np.int32)
        self.history = []
        self.stall, self.prev, self.done = 0, 0.0, False

    def _stats(self, migration=False):
        b = int(np.argmax(self.L))
        self.history.append(float(self.L[b]))
        if self.L[b] > self.best_ever:
            self.best_ever = float(self.L[b])
            self.best_labels = self.pop[b].copy()
        # termination (Q28 for islands: the stall test runs at migration
        # generations only, on the island's post-import best, which is the
        # global best; Q16 for one island)
        best = float(self.L[b])
        if self.G == 1:
            if self.gen > 0:
                self.stall = self.stall + 1 if best - self.prev < self.p.tol else 0
            self.prev = best
        elif migration:
            if self.gen + 1 > self.p.migrate_every:
                self.stall = self.stall + self.p.migrate_every if best - self.prev < self.p.tol else 0
            self.prev = best
        if (self.p.tol >= 0 and self.stall >= self.p.stall_gens) or self.gen + 1 >= self.p.max_gens:
            self.done = True

    def gen_evaluate(self):
        self.L, self.top = orc.evaluate(self.C, self.pop)
        mig = self.G > 1 and (self.gen + 1) % self.p.migrate_every == 0
        if not mig:
            self._stats()
        return mig

    def migrant_bytes(self):
        return self.rec * self.p.migrants

    def export_migrants(self, send):
        order = orc.order(self.L)
        buf = np.zeros(self.migrant_bytes(), np.uint8)
        for r in range(self.p.migrants):
            i = order[r]
            rec = buf[r * self.rec:(r + 1) * self.rec]
            rec[0:8] = np.frombuffer(np.float64(self.L[i]).tobytes(), np.uint8)
            t = 0xFFFF if self.top[i] < 0 else int(self.top[i])
            rec[8:10] = np.frombuffer(np.uint16(t).tobytes(), np.uint8)
            rec[16:16 + 2 * self.N] = np.frombuffer(self.pop[i].astype(np.uint16).tobytes(), np.uint8)
        send.copy_(torch.from_numpy(buf))

    def import_migrants(self, recv, n_islands):
        buf = recv.numpy()
        Em = self.p.migrants
        cands = []
        for j in range(n_islands * Em):
            rec = buf[j * self.rec:(j + 1) * self.rec]
            L = float(np.frombuffer(rec[0:8].tobytes(), np.float64)[0])
            t = int(np.frombuffer(rec[8:10].tobytes(), np.uint16)[0])
            lab = np.frombuffer(rec[16:16 + 2 * self.N].tobytes(), np.uint16).astype(np.int32)
            cands.append((L, -1 if t == 0xFFFF else t, lab))
        used = [False] * len(cands)
        chosen = []
        for _ in range(Em):           # (L desc, island asc, rank asc): strict '>' scan
            b = -1
            for j, c in enumerate(cands):
                if not used[j] and (b < 0 or c[0] > cands[b][0]):
                    b = j
            used[b] = True
            chosen.append(cands[b])
        order = orc.order(self.L)
        for r, (L, t, lab) in enumerate(chosen):
            w = order[self.P - 1 - r]
            self.pop[w] = lab
            self.L[w] = L
            self.top[w] = t
        self._stats(migration=True)

    def gen_breed(self):
        if self.done:                       # the device breed is a no-op once done
            return
        self.pop = orc.step(self.p, self.pop, self.L, self.top, self.gen, island=self.island,
                            p_off=self.island * self.P)
        self.gen += 1

    def state(self):
        return dict(generation=self.gen, best_L=self.best_ever, best_labels=self.best_labels + 1,
                    done=int(self.done))


class OracleReplica:
    """Oracle-backed replica (TEST INFRASTRUCTURE) with the interface of
    paper_1403_4099_b200.replicated.GpuReplica: holds the whole population,
    evaluates only the requested shard, installs gathered fitness, breeds
    with orc_step.  Labels, L and top travel exactly as libpga.so exchanges
    them (fp64 L, 16-bit top with 0xFFFF = none)."""

    def __init__(self, C, params):
        self.C = np.ascontiguousarray(C, np.float64)
        self.N = self.C.shape[0]
        self.p = params
        self.P = params.pop
        self.device = torch.device("cpu")

    def init(self, seed):
        self.p.seed = seed
        self.pop = orc.init_population(seed, self.N, self.P)
        self.gen = 0
        self.best_ever = -1.0
        self.best_labels = np.zeros(self.N, np.int32)
        self.history = []
        self.evaluated = 0

    def rep_evaluate(self, begin, end, L_out, top_out):
        L, top = orc.evaluate(self.C, self.pop[begin:end])
        self.evaluated += end - begin
        L_out.copy_(torch.from_numpy(L))
        top_out.copy_(torch.from_numpy(np.where(top < 0, -1, top).astype(np.int16)))

    def rep_commit(self, L, top):
        self.L = L.numpy().copy()
        t = top.numpy().astype(np.int32)
        self.top = np.where(t == -1, -1, t & 0xFFFF)
        b = int(np.argmax(self.L))
        self.history.append(float(self.L[b]))
        if self.L[b] > self.best_ever:
            self.best_ever = float(self.L[b])
            self.best_labels = self.pop[b].copy()

    def gen_breed(self):
        self.pop = orc.step(self.p, self.pop, self.L, self.top, self.gen)
        self.gen += 1
