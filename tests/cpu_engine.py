"""CPU stand-in for distributed.GpuEngine — test infrastructure only.

Lets the -m "not gpu" suite drive the sharded drivers' collective logic
(gloo, world size 2-3) with a plain union-find that follows the same rules
as the GPU engine: larger root under smaller, each undirected edge of a row
shard processed only as (u, t) with t < u, merging edges recorded."""
from __future__ import annotations

import numpy as np
import torch


def _find(p, x):
    r = x
    while p[r] != r:
        r = p[r]
    while p[x] != r:
        p[x], x = r, p[x]
    return r


def _union(p, u, v):
    a, b = _find(p, u), _find(p, v)
    if a == b:
        return False
    if a < b:
        a, b = b, a
    p[a] = b
    return True


class CpuEngine:
    device = "cpu"

    def local_forest(self, shard, spec):
        n = shard.n
        p = np.arange(n, dtype=np.int64)
        off, tgt = shard.offsets, shard.targets
        fu, fv = [], []
        for u in range(n):
            for j in range(off[u], off[u + 1]):
                t = int(tgt[j])
                if t < u and _union(p, u, t):
                    fu.append(u)
                    fv.append(t)
        return (torch.from_numpy(p.astype(np.int32)), torch.tensor(fu, dtype=torch.int32),
                torch.tensor(fv, dtype=torch.int32))

    def union_list(self, parent, us, vs, spec):
        p = parent.numpy().astype(np.int64)
        mu, mv = [], []
        for u, v in zip(us.tolist(), vs.tolist()):
            if _union(p, u, v):
                mu.append(u)
                mv.append(v)
        parent.copy_(torch.from_numpy(p.astype(np.int32)))
        return torch.tensor(mu, dtype=torch.int32), torch.tensor(mv, dtype=torch.int32)

    # two-phase sharded pipeline (gc_shard_sample / gc_shard_finish semantics)
    def shard_sample(self, shard, spec, record=True):
        n = shard.n
        p = np.arange(n, dtype=np.int64)
        off, tgt = shard.offsets, shard.targets
        fu, fv = [], []
        insp = 0

        def rec(u, t):
            if _union(p, u, t):
                fu.append(u)
                fv.append(t)
        kind = spec.sample.value
        if kind == "kout":
            for u in range(n):
                take = min(spec.kout_k, int(off[u + 1] - off[u]))
                insp += take
                for j in range(take):
                    rec(u, int(tgt[off[u] + j]))
        elif kind == "hb":
            roots = []
            for v in range(n):
                if off[v + 1] > off[v]:
                    insp += 1
                    first = int(tgt[off[v]])
                    if first < v:
                        rec(v, first)
                    else:
                        roots.append(v)
            for v in roots:
                take = min(spec.hb_edges, int(off[v + 1] - off[v]))
                insp += take
                for j in range(take):
                    rec(v, int(tgt[off[v] + j]))
        return (torch.from_numpy(p.astype(np.int32)), torch.tensor(fu, dtype=torch.int32),
                torch.tensor(fv, dtype=torch.int32), insp)

    def shard_finish(self, shard, spec, parent):
        n = shard.n
        p = parent.numpy().astype(np.int64)
        off, tgt = shard.offsets, shard.targets
        lab = np.array([_find(p, v) for v in range(n)], dtype=np.int64)
        fu, fv = [], []
        insp = 0
        if spec.sample.value == "none":
            lmax, cnt, active = n, (1 if n else 0), n
            for u in range(n):
                for j in range(off[u], off[u + 1]):
                    insp += 1
                    t = int(tgt[j])
                    if t < u and _union(p, u, t):
                        fu.append(u)
                        fv.append(t)
        else:
            counts = np.bincount(lab, minlength=n)
            lmax = int(counts.argmax()) if n else 0
            cnt = int(counts[lmax]) if n else 0
            act = np.flatnonzero(lab != lmax)
            active = len(act)
            for u in act.tolist():
                for j in range(off[u], off[u + 1]):
                    insp += 1
                    t = int(tgt[j])
                    if _union(p, u, t):
                        fu.append(u)
                        fv.append(t)
        parent.copy_(torch.from_numpy(p.astype(np.int32)))
        return (torch.tensor(fu, dtype=torch.int32), torch.tensor(fv, dtype=torch.int32),
                {"insp_finish": insp, "l_max": lmax, "lmax_count": cnt, "n_active": active})

    # compact summary exchange (gc_shard_summary / gc_shard_join semantics)
    def shard_summary(self, parent, hint=None, pairs=True):
        p = parent.numpy().astype(np.int64)
        n = len(p)
        lab = np.array([_find(p, v) for v in range(n)], dtype=np.int64)
        if hint is not None:
            g = int(lab[int(hint.item())])
        else:
            g = int(np.bincount(lab, minlength=n).argmax()) if n else 0
        in_g = lab == g
        nw = max((n + 31) // 32, 1)
        bits = np.zeros(nw * 32, dtype=bool)
        bits[:n] = in_g
        words = np.packbits(bits, bitorder="little").view(np.uint32).view(np.int32)
        parent.copy_(torch.from_numpy(lab.astype(np.int32)))
        if not pairs:
            return torch.from_numpy(words.copy()), torch.tensor([g], dtype=torch.int64), None, None
        pair = (~in_g) & (lab != np.arange(n))
        return (torch.from_numpy(words.copy()), torch.tensor([g], dtype=torch.int64),
                torch.from_numpy(np.flatnonzero(pair).astype(np.int32)), torch.from_numpy(lab[pair].astype(np.int32)))

    @staticmethod
    def _classes(words_all, labels_all, n):
        W = words_all.numpy().view(np.uint32)
        R = W.shape[0]
        bits = np.unpackbits(W.view(np.uint8).reshape(R, -1), axis=1, bitorder="little")[:, :n].astype(bool)
        labels = labels_all.numpy()
        par = list(range(R))

        def root(x):
            while par[x] != x:
                x = par[x]
            return x
        for r in range(R):
            for s in range(r + 1, R):
                if (bits[r] & bits[s]).any():
                    a, b = root(r), root(s)
                    if a != b:
                        par[max(a, b)] = min(a, b)
        rep = [min(int(labels[s]) for s in range(R) if root(s) == root(r)) for r in range(R)]
        return bits, rep

    def shard_absorb(self, parent, words_all, labels_all):
        p = parent.numpy().astype(np.int64)
        n = len(p)
        bits, rep = self._classes(words_all, labels_all, n)
        for v in range(n):
            for r in range(len(rep)):
                if bits[r, v]:
                    _union(p, v, rep[r])
                    break
        parent.copy_(torch.from_numpy(p.astype(np.int32)))
        return torch.tensor([rep[0]], dtype=torch.int32)

    def shard_join(self, parent, words_all, labels_all, us, vs, spec):
        n = parent.numel()
        bits, rep = self._classes(words_all, labels_all, n)
        p = np.arange(n, dtype=np.int64)
        for v in range(n):
            for r in range(len(rep)):
                if bits[r, v]:
                    p[v] = rep[r]
                    break
        for u, v in zip(us.tolist(), vs.tolist()):
            _union(p, u, v)
        parent.copy_(torch.from_numpy(p.astype(np.int32)))

    def union_pairs(self, parent, us, vs, spec):
        self.union_list(parent, us, vs, spec)

    def finalize(self, parent, inplace=False):
        p = parent.numpy().astype(np.int64)
        return torch.from_numpy(np.array([_find(p, v) for v in range(len(p))], dtype=np.int32))

    # incremental: parent with sentinel `cap` for uninitialised slots
    def incr_create(self, spec, cap):
        return {"p": np.full(cap, cap, dtype=np.int64), "cap": cap}

    def _init(self, h, x):
        if h["p"][x] == h["cap"]:
            h["p"][x] = x

    def incr_insert_list(self, h, us, vs):
        mu, mv = [], []
        for u, v in zip(us.tolist(), vs.tolist()):
            self._init(h, u)
            self._init(h, v)
            if _union(h["p"], u, v):
                mu.append(u)
                mv.append(v)
        return torch.tensor(mu, dtype=torch.int32), torch.tensor(mv, dtype=torch.int32)

    def incr_insert(self, h, us, vs):
        self.incr_insert_list(h, us, vs)

    def incr_query(self, h, us, vs):
        p, cap = h["p"], h["cap"]

        def root(x):
            return x if p[x] == cap else _find(p, x)
        return torch.tensor([int(root(u) == root(v)) for u, v in zip(us.tolist(), vs.tolist())], dtype=torch.uint8)

    def incr_labels(self, h):
        p, cap = h["p"], h["cap"]
        inited = p != cap
        lab = np.array([_find(p, v) if inited[v] else v for v in range(cap)], dtype=np.int32)
        comps = int(sum(1 for v in range(cap) if inited[v] and lab[v] == v))
        return torch.from_numpy(lab), comps

    # distributed BFS (gc_dbfs_* semantics): int32 bitmap words, as the GPU
    # engine, so the driver's SUM all-reduce of next-frontier words is tested
    @staticmethod
    def _words(n):
        return torch.zeros(max((n + 31) // 32, 1), dtype=torch.int32)

    @staticmethod
    def _test(words, x):
        return bool((int(words[x >> 5]) >> (x & 31)) & 1)

    @staticmethod
    def _set(words, x):
        w = np.array([int(words[x >> 5])], dtype=np.int32).view(np.uint32)
        w |= np.uint32(1 << (x & 31))
        words[x >> 5] = int(w.view(np.int32)[0])

    def dbfs_init(self, n, source):
        st = {"n": n, "F": self._words(n), "V": self._words(n), "M": self._words(n), "N": self._words(n),
              "par": np.full(max(n, 1), -1, dtype=np.int64)}
        self._set(st["F"], source)
        self._set(st["V"], source)
        st["par"][source] = -2
        return st

    def dbfs_marks(self, shard, st):
        lo, hi = getattr(shard, "row_block", (0, shard.n))
        off, tgt = shard.offsets, shard.targets
        st["M"].zero_()
        for f in range(lo, hi):
            if self._test(st["F"], f):
                for j in range(off[f], off[f + 1]):
                    x = int(tgt[j])
                    if not self._test(st["V"], x):
                        self._set(st["M"], x)
        ids = [x for x in range(st["n"]) if self._test(st["M"], x)]
        return torch.tensor(ids, dtype=torch.int32)

    def dbfs_merge_marks(self, st, ids):
        for x in ids.tolist():
            self._set(st["M"], x)

    def dbfs_claim(self, shard, st, marks, foreign=None):
        if foreign is not None:
            self.dbfs_merge_marks(st, foreign)
        lo, hi = getattr(shard, "row_block", (0, shard.n))
        off, tgt = shard.offsets, shard.targets
        st["N"].zero_()
        for x in range(lo, hi):
            if self._test(st["V"], x) or (marks and not self._test(st["M"], x)):
                continue
            for j in range(off[x], off[x + 1]):
                t = int(tgt[j])
                if self._test(st["F"], t):
                    st["par"][x] = t
                    self._set(st["N"], x)
                    break
        return st["N"]

    def dbfs_advance(self, st):
        nw = st["N"].numpy().view(np.uint32)
        st["F"].copy_(st["N"])
        v = st["V"].numpy().view(np.uint32)
        v |= nw
        return int(sum(bin(int(w)).count("1") for w in nw))

    def dbfs_finish(self, shard, st):
        n = st["n"]
        lo, hi = getattr(shard, "row_block", (0, n))
        off = shard.offsets
        reached = [self._test(st["V"], v) for v in range(n)]
        mn = min(v for v in range(n) if reached[v])
        lab = np.array([mn if reached[v] else v for v in range(n)], dtype=np.int32)
        fu, fv, insp = [], [], 0
        for v in range(lo, hi):
            if reached[v]:
                insp += int(off[v + 1] - off[v])
                if st["par"][v] >= 0:
                    fu.append(int(st["par"][v]))
                    fv.append(v)
        return (torch.from_numpy(lab), torch.tensor(fu, dtype=torch.int32), torch.tensor(fv, dtype=torch.int32),
                insp)

    def row_degrees(self, shard, ids):
        off = shard.offsets
        ids = np.asarray(ids, dtype=np.int64)
        return torch.from_numpy((off[ids + 1] - off[ids]).astype(np.int64))
