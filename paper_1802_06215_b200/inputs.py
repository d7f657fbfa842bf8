"""Seeded synthetic inputs for the batched leaf expansion.

This module is shared by the tests, the bench and the oracle legs.  It holds
none of the method's arithmetic: it only draws the paper's workloads (initial
beliefs given as K weighted scenarios; model layouts) with numpy's
own generator and encodes them in the state layouts of the model cards
(DESIGN.md §3).  The scenario random numbers phi_t that the method consumes
are NOT drawn here -- each side implements the counter-based stream itself.

Recipe: belief seed = 1000 + config number, layout seed 7,
uniform weights 1/K rounded to fp32 (a non-uniform set is available for
parity tests).
"""
from __future__ import annotations

import numpy as np

# Classic RockSample(7,8) layout (Smith & Simmons 2004; background knowledge,
# not in the reference -- any fixed layout preserves parity).
RS78_ROCKS = [(2, 0), (0, 1), (3, 1), (6, 3), (2, 4), (3, 4), (5, 5), (1, 6)]
RS78_START = (0, 3)

NAV_LANDMARKS_13 = [(2, 3), (6, 2), (10, 3), (2, 9), (6, 10), (10, 9)]


def _fmt_xy(pts):
    return ",".join(f"{x}:{y}" for x, y in pts)


# --------------------------------------------------------------------------
# RockSample / multi-agent RockSample
# --------------------------------------------------------------------------
def rocksample_layout(n: int, m: int, robots: int, layout_seed: int = 7):
    """Rock cells and robot starts.  RockSample(7,8) with one robot uses the
    classic layout; otherwise robot r starts at (0, floor((r+1) n/(R+1))) and
    m distinct rock cells are drawn from the layout seed."""
    if n == 7 and m == 8 and robots == 1:
        return list(RS78_ROCKS), [RS78_START]
    starts = [(0, ((r + 1) * n) // (robots + 1)) for r in range(robots)]
    rng = np.random.Generator(np.random.PCG64(layout_seed))
    cells = rng.permutation(n * n)[:m]
    rocks = [(int(c % n), int(c // n)) for c in cells]
    return rocks, starts


def rocksample_params(n=7, m=8, robots=1, D=20, gamma=0.95, layout_seed=7, extra=""):
    rocks, starts = rocksample_layout(n, m, robots, layout_seed)
    p = (f"n={n} robots={robots} D={D} gamma={gamma} rocks={_fmt_xy(rocks)} "
         f"starts={_fmt_xy(starts)}")
    return (p + " " + extra).strip()


def rocksample_belief(n, m, robots, K, seed, layout_seed=7, rock_p=0.5):
    """word 0: rock-good bitmask (each rock good w.p. 0.5); word 1: 16-bit
    robot cells y*n+x (all scenarios share the known starts)."""
    _, starts = rocksample_layout(n, m, robots, layout_seed)
    rng = np.random.Generator(np.random.PCG64(seed))
    good = (rng.random((K, m)) < rock_p).astype(np.uint32)
    w0 = (good << np.arange(m, dtype=np.uint32)).sum(axis=1).astype(np.uint32)
    w1 = 0
    for r, (x, y) in enumerate(starts):
        w1 |= (y * n + x) << (16 * r)
    states = np.empty((2, K), dtype=np.uint32)
    states[0] = w0
    states[1] = np.uint32(w1)
    return states


# --------------------------------------------------------------------------
# Navigation in a partially known map
# --------------------------------------------------------------------------
def nav_params(n=13, wall_y=None, gates=(3, 9), landmarks=None, goal=None, D=90, gamma=0.95):
    wall_y = n // 2 if wall_y is None else wall_y
    goal = (n // 2, n - 1) if goal is None else goal
    if landmarks is None:
        landmarks = NAV_LANDMARKS_13 if n == 13 else []
    p = f"n={n} wall_y={wall_y} gates={gates[0]},{gates[1]} goal={goal[0]}:{goal[1]} D={D} gamma={gamma}"
    if landmarks:
        p += f" landmarks={_fmt_xy(landmarks)}"
    return p


def nav_unknown_count(n=13, wall_y=None, landmarks=None):
    wall_y = n // 2 if wall_y is None else wall_y
    if landmarks is None:
        landmarks = NAV_LANDMARKS_13 if n == 13 else []
    rows = n - 3  # all rows but the top, the bottom and the wall
    return rows * n - len([1 for (x, y) in landmarks if y not in (0, n - 1, wall_y)])


def nav_belief(K, seed, n=13, wall_y=None, landmarks=None, p_occ=0.1):
    """word 0: start cell on the top row (uniform) | gate<<8 (uniform);
    words 1..: each unknown cell occupied w.p. 0.1."""
    nu = nav_unknown_count(n, wall_y, landmarks)
    words = 1 + (nu + 31) // 32
    rng = np.random.Generator(np.random.PCG64(seed))
    x = rng.integers(0, n, size=K)
    gate = rng.integers(0, 2, size=K)
    occ = rng.random((K, nu)) < p_occ
    states = np.zeros((words, K), dtype=np.uint32)
    states[0] = (x + (gate << 8)).astype(np.uint32)
    for b in range(nu):
        states[1 + b // 32] |= (occ[:, b].astype(np.uint32) << np.uint32(b % 32))
    return states


# --------------------------------------------------------------------------
# Driving among pedestrians
# --------------------------------------------------------------------------
def car_params(peds=20, D=90, gamma=0.95):
    return f"peds={peds} D={D} gamma={gamma}"


def car_belief(K, seed, peds=20, layout_seed=7):
    """Car at x=0, speed level 2; pedestrian positions fixed by the layout
    seed (x in [2,20), y in [-5,5)), observed; only the goals vary per
    scenario (uniform over 4)."""
    lay = np.random.Generator(np.random.PCG64(layout_seed))
    px = (2.0 + 18.0 * lay.random(peds)).astype(np.float32)
    py = (-5.0 + 10.0 * lay.random(peds)).astype(np.float32)
    rng = np.random.Generator(np.random.PCG64(seed))
    goals = rng.integers(0, 4, size=(K, peds)).astype(np.uint64)
    states = np.zeros((4 + 2 * peds, K), dtype=np.uint32)
    states[0] = np.float32(0.0).view(np.uint32)
    states[1] = 2
    g = (goals << (2 * (np.arange(peds, dtype=np.uint64) % 16))).astype(np.uint64)
    states[2] = g[:, : min(peds, 16)].sum(axis=1).astype(np.uint32)
    if peds > 16:
        states[3] = g[:, 16:].sum(axis=1).astype(np.uint32)
    for i in range(peds):
        states[4 + 2 * i] = px[i].view(np.uint32)
        states[5 + 2 * i] = py[i].view(np.uint32)
    return states


# --------------------------------------------------------------------------
# Tiger (test fixture)
# --------------------------------------------------------------------------
def tiger_params(D=10, gamma=0.95):
    return f"D={D} gamma={gamma}"


def tiger_belief(K, seed):
    rng = np.random.Generator(np.random.PCG64(seed))
    return rng.integers(0, 2, size=(1, K)).astype(np.uint32)


# --------------------------------------------------------------------------
def weights(K, seed=None, uniform=True):
    """Uniform 1/K in fp32, or w ∝ 1 + (u>>8) 2^-24 (non-uniform parity set)."""
    if uniform:
        return np.full(K, np.float32(1.0 / K), dtype=np.float32)
    rng = np.random.Generator(np.random.PCG64(seed))
    u = rng.integers(0, 2**32, size=K, dtype=np.uint64)
    w = 1.0 + (u >> np.uint64(8)).astype(np.float64) * 2.0**-24
    return (w / w.sum()).astype(np.float32)


def select_leaves(child_count, child_begin, num_actions, L, root=0):
    """Leaf generator: the root's children sorted by
    (-N_c, action, child ordinal); the first L become the batch's leaves
    (depth 1).  Returns a list of (action, child_ordinal)."""
    items = []
    for a in range(num_actions):
        b, e = int(child_begin[a]), int(child_begin[a + 1])
        for c in range(e - b):
            items.append((-int(child_count[b + c]), a, c))
    items.sort()
    if len(items) < L:
        raise ValueError(f"root has only {len(items)} children, need {L}")
    return [(a, c) for (_, a, c) in items[:L]]


# --------------------------------------------------------------------------
# Configs of BASELINE.json
# --------------------------------------------------------------------------
CONFIGS = {
    1: dict(kind="rocksample", name="rocksample_7_8_K100_root", n=7, m=8, robots=1, K=100, L=1, D=20, root=True),
    2: dict(kind="rocksample", name="mars_15_15_K500_L64", n=15, m=15, robots=2, K=500, L=64, D=20),
    3: dict(kind="nav", name="nav_13_K500_L64", n=13, K=500, L=64, D=90),
    4: dict(kind="car", name="car_20peds_K500_L64", peds=20, K=500, L=64, D=90),
    5: dict(kind="rocksample", name="mars_15_15_sweep_L256", n=15, m=15, robots=2, K=500, L=256, D=20),
}


def car_roots(L, K, peds=20, base_seed=1004):
    """Config 4's batch: L concurrent root beliefs (crowd layouts and goal
    samples differ per root).  At depth >= 1 every car child holds a single
    scenario (the 0.5 m observation grid separates all of them), so a
    batch of L depth-1 leaves would carry L scenarios; the K=500 workload of
    the config is therefore L roots expanded in one launch."""
    out = []
    for j in range(L):
        seed = base_seed + 1000 * j
        out.append((car_belief(K, seed, peds, layout_seed=7 + j), weights(K, seed), seed))
    return out


def config_inputs(cfg: int, K=None, L=None, uniform=True, D=None, peds=None):
    """(kind, params, states_soa, weights, seed, L) of a BASELINE config
    (peds: pedestrian count of the driving config, default 20)."""
    c = dict(CONFIGS[cfg])
    if peds is not None and c["kind"] == "car":
        c["peds"] = peds
    K = c["K"] if K is None else K
    L = c["L"] if L is None else L
    D = c["D"] if D is None else D
    seed = 1000 + cfg
    if c["kind"] == "rocksample":
        params = rocksample_params(c["n"], c["m"], c["robots"], D=D)
        states = rocksample_belief(c["n"], c["m"], c["robots"], K, seed)
    elif c["kind"] == "nav":
        params = nav_params(c["n"], D=D)
        states = nav_belief(K, seed, c["n"])
    elif c["kind"] == "car":
        params = car_params(c["peds"], D=D)
        states = car_belief(K, seed, c["peds"])
    else:
        raise ValueError(c["kind"])
    return c["kind"], params, states, weights(K, seed, uniform), seed, L
