"""Stand-in multi-edge-type LDPC parity-check matrices (seeded socket matching).

The paper's codes use the degree distributions of ref. [WANGRA], built by PEG
("The degree distribution of these three codes are proposed in
[WANGRA]. The parity check matrices are randomly constructed by progressive edge
growth algorithm"); neither is printed.  The stand-ins below reproduce every
structural count of Table 1 exactly at n = 10^6:

* ``r0.1``: nu = 0.1075 x1^2 x2^21 + 0.0175 x1^3 x2^21 + 0.875 x3,
  mu = 0.0075 x1^10 + 0.0175 x1^11 + 0.875 x2^3 x3.
  n=10^6: E = 3,767,500, m = 900,000, 875,000 degree-1 VNs, E_it = 2,892,500.
* ``r0.05``: nu = 0.04 x1^2 x2^34 + 0.03 x1^3 x2^34 + 0.93 x3,
  mu = 0.01 x1^8 + 0.01 x1^9 + 0.41 x2^2 x3 + 0.52 x2^3 x3.
  n=10^6: E = 3,480,000, m = 950,000, 930,000 degree-1 VNs, E_it = 2,550,000.
* ``r0.1de`` (R29): the same Table-1 counts with degrees chosen by density
  evolution (tools/met_de.py) and finite-length runs (tools/met_search.py):
  nu = 0.05 x1^2 x2^21 + 0.0175 x1^3 x2^21 + 0.0575 x1^3 x2^20 + 0.875 x3,
  mu = 0.025 x1^13 + 0.0575 x2^2 x3 + 0.8175 x2^3 x3, built without 4-cycles
  among the active VNs (DE threshold SNR 0.153 vs 0.182 for ``r0.1``).
* ``r0.02`` (R25): nu = 0.02 x1^2 x2^{56|57} + 0.02 x1^3 x2^{56|57} + 0.96 x3,
  mu = 0.02 x1^5 + 0.6025 x2^2 x3 + 0.3575 x2^3 x3 (inner degree 57 on 37,500 of the 40,000
  active VNs).  n=10^6: E = 3,337,500, m = 980,000, 960,000 degree-1 VNs, E_it = 2,377,500.

Construction: per edge type, VN sockets are matched to a seeded Fisher-Yates
shuffle of CN sockets; parallel edges are repaired by random swaps inside the
type; VN and CN labels are then randomly permuted (so the degree-1 VNs are not
a contiguous block), and the matrix is canonicalised: CSR rows ascending in CN
index, each row ascending in VN index; CSC columns ascending in CN index.

A ``Code`` carries the edge-indexed storage the C-ABI takes (BASELINE.json
north_star "stored edge-indexed as CSR plus CSC permutations"): ``cn_ptr[m+1]``,
``edge_vn[E]`` (VN of CSR edge e), ``vn_ptr[n+1]``, ``vn_edge[E]`` (CSR edge id
of CSC slot k).
"""
from __future__ import annotations

import dataclasses
import os
from pathlib import Path

import numpy as np

CODE_SEED = 1711
# generated codes are cached outside the repository (a 10^6 code is ~60 MB; the cache is a
# pure function of (family, n, seed) and is rebuilt in seconds when missing)
_CACHE = Path(os.environ.get("METLDPC_CODE_CACHE", Path.home() / ".cache" / "metldpc" / "codes"))


@dataclasses.dataclass
class Code:
    n: int
    m: int
    cn_ptr: np.ndarray   # int64 [m+1]
    edge_vn: np.ndarray  # int32 [E]
    vn_ptr: np.ndarray   # int64 [n+1]
    vn_edge: np.ndarray  # int64 [E]  CSR edge id of CSC slot k
    name: str = "code"

    @property
    def num_edges(self) -> int:
        return int(self.edge_vn.shape[0])

    @property
    def vn_degree(self) -> np.ndarray:
        return np.diff(self.vn_ptr)

    @property
    def cn_degree(self) -> np.ndarray:
        return np.diff(self.cn_ptr)

    def edge_cn(self) -> np.ndarray:
        return np.repeat(np.arange(self.m, dtype=np.int32), self.cn_degree)

    def dense(self) -> np.ndarray:
        h = np.zeros((self.m, self.n), dtype=np.uint8)
        h[self.edge_cn(), self.edge_vn] = 1
        return h

    def stats(self) -> dict:
        vd = self.vn_degree
        n1 = int((vd == 1).sum())
        return {
            "n": self.n, "m": self.m, "edges": self.num_edges,
            "n_deg1": n1, "n_active": self.n - n1,
            "iter_edges": self.num_edges - n1,
            "max_cn_deg": int(self.cn_degree.max()), "max_vn_deg": int(vd.max()),
            "rate": (self.n - self.m) / self.n,
        }


def from_edges(n: int, m: int, vn: np.ndarray, cn: np.ndarray, name: str = "code") -> Code:
    """Canonical edge-indexed CSR + CSC from an edge list (no duplicate check)."""
    vn = np.asarray(vn, dtype=np.int64)
    cn = np.asarray(cn, dtype=np.int64)
    order = np.lexsort((vn, cn))          # CSR: by CN, then VN
    vn, cn = vn[order], cn[order]
    cn_ptr = np.zeros(m + 1, dtype=np.int64)
    np.cumsum(np.bincount(cn, minlength=m), out=cn_ptr[1:])
    csc = np.lexsort((cn, vn))            # CSC slots: by VN, then CN (stable over CSR ids)
    vn_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(vn, minlength=n), out=vn_ptr[1:])
    return Code(n=n, m=m, cn_ptr=cn_ptr, edge_vn=vn.astype(np.int32),
                vn_ptr=vn_ptr, vn_edge=csc.astype(np.int64), name=name)


def from_dense(h: np.ndarray, name: str = "dense") -> Code:
    h = np.asarray(h)
    cn, vn = np.nonzero(h)
    return from_edges(h.shape[1], h.shape[0], vn, cn, name=name)


# ----------------------------------------------------------------------------- MET stand-ins

def met_counts(family: str, n: int) -> dict:
    """Node/edge counts of the stand-in ensemble at length n."""
    if family == "r0.1":
        if n % 8:
            raise ValueError("r0.1 stand-in needs n divisible by 8")
        a = n // 8
        a3 = int(round(0.14 * a))
        a2 = a - a3
        n1 = 7 * n // 8
        m = n - int(round(0.1 * n))
        inner = {3: n1}                      # CNs x2^3 x3
        vn_core = {2: a2, 3: a3}
        inner_per_vn = 21
    elif family == "r0.1de":
        # DESIGN.md R29 / SURVEY 8(f) #4: same Table-1 counts (n_1 = 7n/8, m = n - 0.1 n,
        # E_it = 2.8925 n, one degree-1 VN per inner check), degrees chosen by density evolution
        # (tools/met_de.py) and finite-length runs (tools/met_search.py): 0.0575 n inner checks
        # x2^2 x3, the rest x2^3 x3, which leaves exactly 13 x (m - n_1) core edges: every core
        # check has degree 13 (one kernel class); VN core degrees 2/3, inner VN degrees 20/21;
        # no 4-cycles among the active VNs (make_met_code).  DE threshold SNR 0.153 on the
        # BIAWGN channel (r0.1: 0.182).
        if n % 8:
            raise ValueError("r0.1de stand-in needs n divisible by 8")
        a = n // 8
        n1 = 7 * n // 8
        m = n - int(round(0.1 * n))
        t2 = int(round(0.0575 * n))
        inner = {2: t2, 3: n1 - t2}
        e2 = 2 * t2 + 3 * (n1 - t2)
        e1 = int(round(2.8925 * n)) - e2
        a3 = e1 - 2 * a
        if not 0 <= a3 <= a or t2 > n1:
            raise ValueError("r0.1de stand-in infeasible at this n")
        a2 = a - a3
        vn_core = {2: a2, 3: a3}
        lo, n_hi = divmod(e2, a)
        # the inner degree lo + 1 goes to the first n_hi active VNs, i.e. core degree 2 first
        inner_per_vn = np.concatenate([np.full(n_hi, lo + 1), np.full(a - n_hi, lo)])
    elif family == "r0.05":
        a = int(round(0.07 * n))
        a3 = int(round(3 * a / 7))
        a2 = a - a3
        n1 = n - a
        m = n - int(round(0.05 * n))
        k3 = 34 * a - 2 * n1
        k2 = n1 - k3
        if k3 < 0 or k2 < 0:
            raise ValueError("r0.05 stand-in infeasible at this n")
        inner = {2: k2, 3: k3}               # CNs x2^2 x3 and x2^3 x3
        vn_core = {2: a2, 3: a3}
        inner_per_vn = 34
    elif family == "r0.02":
        # Table 1 rate-0.02 column: E_it = 2.3775 n, n_1 = 0.96 n.
        a = int(round(0.04 * n))
        a3 = a // 2
        a2 = a - a3
        n1 = n - a
        m = n - int(round(0.02 * n))
        t2 = int(round(2.3775 * n)) - (2 * a2 + 3 * a3)
        lo, n_hi = divmod(t2, a)
        k3 = t2 - 2 * n1
        k2 = n1 - k3
        if k3 < 0 or k2 < 0 or m - n1 <= 0:
            raise ValueError("r0.02 stand-in infeasible at this n")
        inner = {2: k2, 3: k3}
        vn_core = {2: a2, 3: a3}
        inner_per_vn = np.concatenate([np.full(n_hi, lo + 1), np.full(a - n_hi, lo)])
    else:
        raise ValueError(f"unknown family {family!r}")
    core = m - n1
    e1 = sum(d * c for d, c in vn_core.items())
    lo = e1 // core
    n_hi = e1 - lo * core
    return {"n": n, "m": m, "a2": a2, "a3": a3, "n1": n1, "core": core,
            "core_deg": {lo: core - n_hi, lo + 1: n_hi} if n_hi else {lo: core},
            "inner": inner, "vn_core": vn_core, "inner_per_vn": inner_per_vn,
            "edges": e1 + int(np.sum(np.broadcast_to(inner_per_vn, (a2 + a3,)))) + n1}


def _match(rng, vn_sock: np.ndarray, cn_sock: np.ndarray, m: int):
    """Seeded socket matching + parallel-edge repair by random swaps."""
    cn = cn_sock.copy()
    rng.shuffle(cn)
    vn = vn_sock
    for _ in range(1000):
        key = vn.astype(np.int64) * m + cn
        order = np.argsort(key, kind="stable")
        ks = key[order]
        dup = order[1:][ks[1:] == ks[:-1]]
        if dup.size == 0:
            return vn, cn
        other = rng.integers(0, cn.size, size=dup.size)
        cn[dup], cn[other] = cn[other], cn[dup].copy()
    raise RuntimeError("parallel-edge repair did not converge")


def break_4cycles(vn_all, cn_all, typ, rng, max_rounds=50):
    """Swap check sockets (within an edge type) until no two active VNs share two checks (at
    n = 10^6 two rounds suffice; small codes keep some 4-cycles after max_rounds)."""
    vn_all = vn_all.copy()
    cn_all = cn_all.copy()
    for rnd in range(max_rounds):
        order = np.lexsort((vn_all, cn_all))
        cs, vs = cn_all[order], vn_all[order]
        starts = np.flatnonzero(np.r_[True, cs[1:] != cs[:-1]])
        ends = np.r_[starts[1:], cs.size]
        deg = ends - starts
        # all VN pairs inside each check (vectorised per degree)
        keys, eidx = [], []
        for d in np.unique(deg):
            if d < 2:
                continue
            st = starts[deg == d]
            blk = st[:, None] + np.arange(d)[None, :]
            iu, ju = np.triu_indices(d, 1)
            u, v = vs[blk[:, iu]], vs[blk[:, ju]]
            keys.append((u.astype(np.int64) << 32) | v.astype(np.int64))
            eidx.append(order[blk[:, ju]])
        keys = np.concatenate([k.ravel() for k in keys])
        eidx = np.concatenate([e.ravel() for e in eidx])
        o = np.argsort(keys, kind="stable")
        ks = keys[o]
        dup = o[1:][ks[1:] == ks[:-1]]
        if dup.size == 0:
            return vn_all, cn_all, rnd
        bad = np.unique(eidx[dup])
        # swap each bad edge's check with a random edge of the same type
        for t in np.unique(typ[bad]):
            b = bad[typ[bad] == t]
            pool = np.setdiff1d(np.flatnonzero(typ == t), b)
            if b.size > pool.size // 2:   # small codes: 4-cycles cannot all be removed; swap a subset
                b = rng.choice(b, size=max(pool.size // 2, 0), replace=False)
            if b.size == 0:
                continue
            other = rng.choice(pool, size=b.size, replace=False)   # disjoint from b: a permutation
            cn_all[b], cn_all[other] = cn_all[other], cn_all[b].copy()
        # parallel edges created by swaps: undo by re-swapping randomly next round (checked above
        # as a duplicate pair only between distinct checks, so check them here)
        key = vn_all.astype(np.int64) * (cn_all.max() + 1) + cn_all
        _, first = np.unique(key, return_index=True)
        par = np.setdiff1d(np.arange(key.size), first)
        for e in par:
            t = typ[e]
            pool = np.flatnonzero(typ == t)
            o2 = int(rng.choice(pool))
            cn_all[e], cn_all[o2] = int(cn_all[o2]), int(cn_all[e])
    return vn_all, cn_all, max_rounds


def make_met_code(family: str, n: int, seed: int = CODE_SEED, cache: bool = True) -> Code:
    name = f"{family}_n{n}_s{seed}"
    path = _CACHE / f"{name}.npz"
    if cache and path.exists():
        z = np.load(path)
        return Code(n=int(z["n"]), m=int(z["m"]), cn_ptr=z["cn_ptr"], edge_vn=z["edge_vn"],
                    vn_ptr=z["vn_ptr"], vn_edge=z["vn_edge"], name=name)
    c = met_counts(family, n)
    rng = np.random.Generator(np.random.Philox(key=seed))
    m = c["m"]
    # VN labels before relabelling: [0,a2) core-deg 2, [a2,a) core-deg 3, [a,n) degree-1
    a = c["a2"] + c["a3"]
    core_deg_vn = np.concatenate([np.full(c["a2"], 2), np.full(c["a3"], 3)])
    # CN labels: [0,core) core CNs, [core,m) inner CNs
    cd = sorted(c["core_deg"].items())
    core_deg_cn = np.concatenate([np.full(cnt, d) for d, cnt in cd])
    inner_deg = np.concatenate([np.full(cnt, d) for d, cnt in sorted(c["inner"].items())])
    core_ids = np.arange(c["core"])
    inner_ids = np.arange(c["core"], m)
    # type 1 (core edges)
    v1, c1 = _match(rng, np.repeat(np.arange(a), core_deg_vn), np.repeat(core_ids, core_deg_cn), m)
    # type 2 (inner edges of active VNs)
    v2, c2 = _match(rng, np.repeat(np.arange(a), c["inner_per_vn"]), np.repeat(inner_ids, inner_deg), m)
    if family == "r0.1de":   # no two active VNs share two checks (4-cycles; R29)
        vv, cc, _ = break_4cycles(np.concatenate([v1, v2]), np.concatenate([c1, c2]),
                               np.concatenate([np.ones(v1.size, np.int8), np.full(v2.size, 2, np.int8)]), rng)
        v1, c1, v2, c2 = vv[:v1.size], cc[:v1.size], vv[v1.size:], cc[v1.size:]
    # type 3 (one degree-1 VN per inner CN)
    v3 = np.arange(a, n)
    c3 = rng.permutation(inner_ids)
    vn = np.concatenate([v1, v2, v3])
    cn = np.concatenate([c1, c2, c3])
    pv = rng.permutation(n)
    pc = rng.permutation(m)
    code = from_edges(n, m, pv[vn], pc[cn], name=name)
    if cache:
        _CACHE.mkdir(parents=True, exist_ok=True)
        tmp = path.with_suffix(".tmp.npz")
        np.savez(tmp, n=n, m=m, cn_ptr=code.cn_ptr, edge_vn=code.edge_vn,
                 vn_ptr=code.vn_ptr, vn_edge=code.vn_edge)
        os.replace(tmp, path)
    return code


# ----------------------------------------------------------------------------- small random codes

def random_code(n: int, m: int, rng: np.random.Generator, frac_deg1: float = 0.5,
                act_deg=(2, 3), max_tries: int = 200) -> Code:
    """Small random code with a given share of degree-1 VNs (tests only).

    Every VN has degree >= 1, no duplicate edges; CN degrees are whatever the
    random placement gives (>= 1 guaranteed by construction).
    """
    for _ in range(max_tries):
        n1 = int(round(frac_deg1 * n))
        deg = np.concatenate([np.ones(n1, int), rng.integers(act_deg[0], act_deg[1] + 1, n - n1)])
        deg = np.minimum(deg, m)
        rng.shuffle(deg)
        h = np.zeros((m, n), np.uint8)
        for v in range(n):
            h[rng.choice(m, size=deg[v], replace=False), v] = 1
        if (h.sum(1) >= 1).all():
            return from_dense(h, name=f"rand_n{n}_m{m}")
    raise RuntimeError("could not draw a code with every CN connected")


def tree_code(rng: np.random.Generator, n_cn: int = 4, cn_deg=(2, 4)) -> Code:
    """Cycle-free Tanner graph (a tree) built by attaching CNs one at a time.

    Each new CN attaches to exactly one existing VN and brings fresh VNs, so
    the factor graph stays a tree and BP is exact (textbook result).
    """
    edges = []
    n = 0
    for j in range(n_cn):
        d = int(rng.integers(cn_deg[0], cn_deg[1] + 1))
        if j == 0:
            vs = list(range(d))
            n = d
        else:
            anchor = int(rng.integers(0, n))
            vs = [anchor] + list(range(n, n + d - 1))
            n += d - 1
        edges += [(v, j) for v in vs]
    vn = np.array([e[0] for e in edges])
    cn = np.array([e[1] for e in edges])
    return from_edges(n, n_cn, vn, cn, name=f"tree_{n}")


# ----------------------------------------------------------------------------- alist I/O

def write_alist(code: Code, path) -> None:
    """MacKay alist: 'n m', 'max_vn max_cn', VN degrees, CN degrees, 1-based lists."""
    vd, cd = code.vn_degree, code.cn_degree
    edge_cn = code.edge_cn()
    lines = [f"{code.n} {code.m}", f"{vd.max()} {cd.max()}",
             " ".join(map(str, vd)), " ".join(map(str, cd))]
    for v in range(code.n):
        sl = code.vn_edge[code.vn_ptr[v]:code.vn_ptr[v + 1]]
        lines.append(" ".join(str(int(edge_cn[e]) + 1) for e in sl))
    for j in range(code.m):
        lines.append(" ".join(str(int(x) + 1) for x in code.edge_vn[code.cn_ptr[j]:code.cn_ptr[j + 1]]))
    Path(path).write_text("\n".join(lines) + "\n")
