"""Weapon-target assignment scenarios (proj/include/gmpea/wta.hpp, wta.cpp):
built-in P1..P10, the scenario file format, and the problem wrapper — so
large synthetic instances can be loaded into the engine."""
from __future__ import annotations

import ctypes as C
import dataclasses
from typing import List

import numpy as np

from . import _lib as g


@dataclasses.dataclass
class WTAInstance:
    """wta.hpp:17-28; p[i][k] is the interception probability of strike k on target i."""

    scenario: str
    n_targets: int
    n_vehicles: int
    max_strikes: List[int]
    p: List[List[float]]
    capacity: List[int]

    def total_slots(self) -> int:
        return int(sum(self.max_strikes))

    def gene_count(self) -> int:
        return self.total_slots() * self.n_vehicles

    def gene_index(self, i: int, k: int, m: int) -> int:
        """Flat slot-major index (wta.cpp:17-21)."""
        return (sum(self.max_strikes[:i]) + k) * self.n_vehicles + m


WTA_MAX_SYNTHETIC = 123  # 3 + 122 // 2 = 64 vehicles, the engine's limit


def wta_scenario(id: str) -> WTAInstance:
    """Built-in scenarios P1..P10 (wta.cpp:23-49), identical tables."""
    if len(id) < 2 or id[0] != "P" or not id[1:].isdigit() or not 1 <= int(id[1:]) <= 10:
        raise ValueError("unknown WTA scenario: " + id)
    return _scenario(int(id[1:]))


def wta_synthetic(num: int) -> WTAInstance:
    """Large synthetic instances: the reference's
    scenario formula (wta.cpp:31-46: 4 + 2(num - 1) targets, 3 + (num - 1)/2
    vehicles, 1-3 strikes, capacity 2-4, probabilities from the seeded
    mt19937_64 stream) continued past P10, where the reference stops.  Equal
    to wta_scenario for num <= 10."""
    if not 1 <= int(num) <= WTA_MAX_SYNTHETIC:
        raise ValueError(f"unknown WTA scenario: P{num}")
    return _scenario(int(num))


def _scenario(num: int) -> WTAInstance:
    nt, nv = 4 + 2 * (num - 1), 3 + (num - 1) // 2
    t, v = C.c_int32(), C.c_int32()
    strikes = np.zeros(nt, np.int32)
    cap = np.zeros(nv, np.int32)
    pr = np.zeros(3 * nt)
    g._check(g._L.gmpea_wta_scenario(num, C.byref(t), C.byref(v), strikes.ctypes.data_as(g._i32p),
                                     cap.ctypes.data_as(g._i32p), pr.ctypes.data_as(g._dp)))
    id = f"P{num}"
    s = strikes[:t.value].tolist()
    p, o = [], 0
    for k in s:
        p.append(pr[o:o + k].tolist())
        o += k
    return WTAInstance(id, t.value, v.value, s, p, cap[:v.value].tolist())


def save_wta(inst: WTAInstance, path: str) -> None:
    """wta.cpp:131-146 (probabilities with 17 significant digits)."""
    with open(path, "w") as f:
        f.write(f"scenario {inst.scenario}\ntargets {inst.n_targets}\nvehicles {inst.n_vehicles}\n")
        f.write("strikes" + "".join(f" {s}" for s in inst.max_strikes) + "\n")
        f.write("capacity" + "".join(f" {c}" for c in inst.capacity) + "\n")
        for i in range(inst.n_targets):
            for k in range(inst.max_strikes[i]):
                f.write(f"p {i} {k} {inst.p[i][k]:.17g}\n")


def load_wta(path: str) -> WTAInstance:
    """wta.cpp:148-192, same validation messages."""
    try:
        lines = open(path).read().splitlines()
    except OSError:
        raise RuntimeError("load_wta: cannot open " + path)
    scen, nt, nv, strikes, cap, p = "", 0, 0, [], [], []
    for line in lines:
        tok = line.split()
        if not tok:
            continue
        key = tok[0]
        if key == "scenario":
            scen = tok[1] if len(tok) > 1 else ""
        elif key == "targets":
            nt = int(tok[1])
        elif key == "vehicles":
            nv = int(tok[1])
        elif key == "strikes":
            strikes += [int(x) for x in tok[1:]]
        elif key == "capacity":
            cap += [int(x) for x in tok[1:]]
        elif key == "p":
            i, k, prob = int(tok[1]), int(tok[2]), float(tok[3])
            while len(p) <= i:
                p.append([])
            while len(p[i]) <= k:
                p[i].append(0.0)
            p[i][k] = prob
        else:
            raise RuntimeError(f"load_wta: unknown key '{key}' in {path}")
    if nt == 0 or nv == 0 or len(strikes) != nt or len(cap) != nv or len(p) != nt:
        raise RuntimeError("load_wta: incomplete scenario in " + path)
    for i in range(nt):
        if len(p[i]) != strikes[i]:
            raise RuntimeError("load_wta: probability table mismatch in " + path)
        if any(not (0.0 <= v <= 1.0) for v in p[i]):
            raise RuntimeError("load_wta: probability out of range in " + path)
    return WTAInstance(scen, nt, nv, strikes, p, cap)


def make_wta_problem(inst: WTAInstance) -> g.Problem:
    """make_wta_problem (wta.cpp:112-129): genes in [0, 1], f = (-interception, ammunition)."""
    flat = [v for row in inst.p for v in row]
    return g.make_wta_problem(inst.scenario, inst.n_targets, inst.n_vehicles, inst.max_strikes, inst.capacity, flat)
