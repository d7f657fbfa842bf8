"""Pins of the oracle's default policies pi0, upper-bound
heuristics u(phi) (Eq. 11) and the driving heading noise.

These parts are PROPOSED by the model cards,
so the pins are hand traces and closed forms worked out from the cards
(not from the oracle's code), a brute-force shortest path, and statistics:

* RockSample(7,8) and a custom 5x5 instance: whole roll-outs traced by hand
  -- the exact action list (FNV-1a hash), length and return -- on streams
  whose sensing outcomes are selected from the pinned Philox words and the
  closed-form thresholds T(p) of the card's accuracy curve (R17);
* a two-robot MARS roll-out traced by hand (joint actions a = b0 + (5+m) b1);
* navigation pi0 over every branch (S, SE, SW, E/W by depth parity, STAY);
* RockSample/MARS u(s) in closed form (one good rock at distance d:
  10 g^d + 10 g^(n-1-x); two robots: the nearer one; exited robots drop out);
* navigation u(s) = 20 g^(d-1) with d the BFS distance to the goal on the
  obstacle-free 8-connected grid whose wall row is open only at the gate
  (every cell of the 13x13 and 5x5 maps, both gates);
* the heading-noise angle: mean 0 and standard deviation pi/8 +- 2 % over
  10^5 draws (the card's sigma; "Gaussian noises on their heading
  directions"), symmetric, bounded.
"""
import math
from collections import deque

import numpy as np
import pytest

import oracle
from paper_1802_06215_b200 import inputs

GAMMA = 0.95
FNV_OFFSET, FNV_PRIME = 0xCBF29CE484222325, 0x100000001B3


def fnv(actions):
    h = FNV_OFFSET
    for a in actions:
        h = ((h ^ a) * FNV_PRIME) & 0xFFFFFFFFFFFFFFFF
    return h


def word(seed, sid, t, k):
    """word k of scenario sid's random numbers at depth t (R13), from the
    Philox block pinned by the known-answer vectors"""
    return int(oracle.philox([sid, t, k // 4, 0], [seed & 0xFFFFFFFF, seed >> 32])[k % 4])


def correct(u, d2):
    """the card's sensing event: correct iff u < T(0.5 (1 + 2^(-sqrt(d2)/4)))"""
    p = 0.5 * (1.0 + 2.0 ** (-math.sqrt(d2) / 4.0))
    return u < (2**32 if p >= 1.0 else math.floor(p * 2**32))


def rs_state(n, good_mask, cells):
    w1 = 0
    for r, c in enumerate(cells):
        w1 |= (0xFFFF if c is None else c[1] * n + c[0]) << (16 * r)
    return np.array([good_mask, w1], np.uint32)


def find_id(seed, depth, wants, max_ids=5000):
    """first scenario id whose sensing words give the wanted outcomes;
    wants: [(step k of the roll-out, robot r, squared distance, correct?)];
    step k from depth `depth` draws phi at depth depth + k + 1"""
    for sid in range(max_ids):
        if all(correct(word(seed, sid, depth + k + 1, r), d2) == want for (k, r, d2, want) in wants):
            return sid
    raise AssertionError("no stream with the wanted readings")


def check_trace(m, s, seed, sid, depth, actions, ret):
    got_ret, got_len, got_hash, _ = m.rollout(s, None, sid, depth, seed)
    assert got_len == len(actions), (got_len, actions)
    assert got_hash == fnv(actions), actions
    assert abs(got_ret - ret) <= 1e-12 * max(1.0, abs(ret)), (got_ret, ret)


# ----------------------------------------------------------------------------
# RockSample(7,8): rocks (2,0) (0,1) (3,1) (6,3) (2,4) (3,4) (5,5) (1,6), start
# (0,3).  Robot 0 handles every rock, sorted by (x, y, j): 1, 7, 0, 4, 2, 5, 6, 3.
# Sub-actions 0 N, 1 S, 2 E, 3 W, 4 SAMPLE, 5 + j SENSE j.
# ----------------------------------------------------------------------------
RS78 = inputs.RS78_ROCKS
ORDER78 = [1, 7, 0, 4, 2, 5, 6, 3]


def d2(p, j, rocks=RS78):
    return (p[0] - rocks[j][0]) ** 2 + (p[1] - rocks[j][1]) ** 2


def test_rs78_trace_sense_good_walk_north_sample_then_sense_rest_and_exit():
    """Rock 1 good, read GOOD (correct) from (0,3): N, N to (0,1), SAMPLE +10;
    the other seven rocks read BAD (correct) from (0,1) in the policy order
    and are dropped; then E seven times, the last one exits (+10)."""
    m = oracle.Model("rocksample", inputs.rocksample_params())
    seed, depth = 1001, 1
    rest = ORDER78[1:]
    wants = [(0, 0, d2((0, 3), 1), True)] + [(4 + i, 0, d2((0, 1), j), True) for i, j in enumerate(rest)]
    sid = find_id(seed, depth, wants)
    actions = [5 + 1, 0, 0, 4] + [5 + j for j in rest] + [2] * 7
    assert actions[:11] == [6, 0, 0, 4, 12, 5, 9, 7, 10, 11, 8]
    check_trace(m, rs_state(7, 1 << 1, [(0, 3)]), seed, sid, depth, actions, 10 * GAMMA**3 + 10 * GAMMA**17)


def test_rs78_trace_wrong_good_reading_samples_a_bad_rock():
    """All rocks bad, rock 1 read GOOD (a wrong reading): the robot walks to
    it and SAMPLEs for -10; the rest read BAD (correct); exit at step 17."""
    m = oracle.Model("rocksample", inputs.rocksample_params())
    seed, depth = 77, 1
    rest = ORDER78[1:]
    wants = [(0, 0, d2((0, 3), 1), False)] + [(4 + i, 0, d2((0, 1), j), True) for i, j in enumerate(rest)]
    sid = find_id(seed, depth, wants)
    actions = [6, 0, 0, 4] + [5 + j for j in rest] + [2] * 7
    check_trace(m, rs_state(7, 0, [(0, 3)]), seed, sid, depth, actions, -10 * GAMMA**3 + 10 * GAMMA**17)


def test_rs78_trace_bad_reading_drops_rock_then_x_first_moves():
    """Rock 1 bad and read BAD: dropped at once.  Rock 7 at (1,6) good and
    read GOOD from (0,3): E first (x before y), then S three times, SAMPLE
    +10 at step 6; the remaining six rocks read BAD from (1,6); E five times
    to x = 6 and the exit at step 18 (19 steps: exactly D - depth)."""
    m = oracle.Model("rocksample", inputs.rocksample_params())
    seed, depth = 2024, 1
    rest = ORDER78[2:]
    wants = [(0, 0, d2((0, 3), 1), True), (1, 0, d2((0, 3), 7), True)]
    wants += [(7 + i, 0, d2((1, 6), j), True) for i, j in enumerate(rest)]
    sid = find_id(seed, depth, wants)
    actions = [6, 12, 2, 1, 1, 1, 4] + [5 + j for j in rest] + [2] * 6
    assert len(actions) == 19
    check_trace(m, rs_state(7, 1 << 7, [(0, 3)]), seed, sid, depth, actions, 10 * GAMMA**6 + 10 * GAMMA**18)


def test_rs_trace_west_and_north_moves_on_a_custom_map():
    """5x5, rocks (1,1) and (3,4), start (4,2), both good, readings correct:
    SENSE 0, W W W, N, SAMPLE (+10), SENSE 1, E E, S S S, SAMPLE (+10), E, E
    (exit +10)."""
    rocks = [(1, 1), (3, 4)]
    params = "n=5 robots=1 D=30 gamma=0.95 rocks=1:1,3:4 starts=4:2"
    m = oracle.Model("rocksample", params)
    seed, depth = 5, 2
    wants = [(0, 0, d2((4, 2), 0, rocks), True), (6, 0, d2((1, 1), 1, rocks), True)]
    sid = find_id(seed, depth, wants)
    actions = [5, 3, 3, 3, 0, 4, 6, 2, 2, 1, 1, 1, 4, 2, 2]
    check_trace(m, rs_state(5, 0b11, [(4, 2)]), seed, sid, depth, actions,
                10 * GAMMA**5 + 10 * GAMMA**12 + 10 * GAMMA**14)


def test_rs_trace_truncated_at_depth_D():
    """The same custom roll-out started at depth 20 with D = 30 stops after
    10 steps (tail l = 0): only the first SAMPLE is collected."""
    rocks = [(1, 1), (3, 4)]
    params = "n=5 robots=1 D=30 gamma=0.95 rocks=1:1,3:4 starts=4:2"
    m = oracle.Model("rocksample", params)
    seed, depth = 5, 20
    wants = [(0, 0, d2((4, 2), 0, rocks), True), (6, 0, d2((1, 1), 1, rocks), True)]
    sid = find_id(seed, depth, wants)
    actions = [5, 3, 3, 3, 0, 4, 6, 2, 2, 1]
    check_trace(m, rs_state(5, 0b11, [(4, 2)]), seed, sid, depth, actions, 10 * GAMMA**5)


def test_mars_two_robot_trace():
    """MARS 5x5, m = 4: rocks j0 (2,1), j1 (1,4), j2 (3,0), j3 (3,3); robot 0
    at (0,1) handles j0, j2; robot 1 at (0,3) handles j1, j3; all good and
    read GOOD.  Joint action a = b0 + 9 b1.  Traced by hand:
      0 SENSE j0 | SENSE j1      6 N (3,0)     | E (3,4)
      1 E (1,1)  | E (1,3)       7 SAMPLE +10  | N (3,3)
      2 E (2,1)  | S (1,4)       8 E (4,0)     | SAMPLE +10
      3 SAMPLE +10 | SAMPLE +10  9 E exit +10  | E (4,3)
      4 SENSE j2 | SENSE j3     10 E (no-op)   | E exit +10 -> terminal
      5 E (3,1)  | E (2,4)"""
    rocks = [(2, 1), (1, 4), (3, 0), (3, 3)]
    params = "n=5 robots=2 D=20 gamma=0.95 rocks=2:1,1:4,3:0,3:3 starts=0:1,0:3"
    m = oracle.Model("rocksample", params)
    assert m.A == 81
    seed, depth = 31, 1
    wants = [(0, 0, d2((0, 1), 0, rocks), True), (0, 1, d2((0, 3), 1, rocks), True),
             (4, 0, d2((2, 1), 2, rocks), True), (4, 1, d2((1, 4), 3, rocks), True)]
    sid = find_id(seed, depth, wants)
    b = [(5, 6), (2, 2), (2, 1), (4, 4), (7, 8), (2, 2), (0, 2), (4, 0), (2, 4), (2, 2), (2, 2)]
    actions = [b0 + 9 * b1 for b0, b1 in b]
    assert actions == [59, 20, 11, 40, 79, 20, 18, 4, 38, 20, 20]
    ret = 20 * GAMMA**3 + 10 * GAMMA**7 + 10 * GAMMA**8 + 10 * GAMMA**9 + 10 * GAMMA**10
    check_trace(m, rs_state(5, 0b1111, [(0, 1), (0, 3)]), seed, sid, depth, actions, ret)


def test_mars_policy_rock_split_by_robot_index():
    """Robot r handles the rocks j = r (mod 2): with one rock per robot left
    UNKNOWN each senses its own (not the nearer one)."""
    params = "n=5 robots=2 D=20 gamma=0.95 rocks=0:3,0:1 starts=0:1,0:3"
    m = oracle.Model("rocksample", params)
    # robot 0 at (0,1) stands on rock 1 but handles rock 0 (at (0,3)), robot 1 the reverse
    a = m.default_action(rs_state(5, 0b11, [(0, 1), (0, 3)]), 0, 0, 1)
    assert a == (5 + 0) + 7 * (5 + 1)
    # memory: rock 0 GOOD (01), rock 1 DONE (10) -> robot 0 moves S toward (0,3), robot 1 goes E
    a = m.default_action(rs_state(5, 0b11, [(0, 1), (0, 3)]), 0, 0b1001, 1)
    assert a == 1 + 7 * 2
    # an exited robot takes E
    a = m.default_action(rs_state(5, 0b11, [None, (0, 3)]), 0, 0, 1)
    assert a == 2 + 7 * (5 + 1)


# ----------------------------------------------------------------------------
# RockSample / MARS upper bound (card: 10 g^(min_r |r - j|_1) per good rock
# + 10 g^(n-1-x_r) per active robot)
# ----------------------------------------------------------------------------
def test_rs78_upper_bound_closed_forms():
    m = oracle.Model("rocksample", inputs.rocksample_params())
    g = GAMMA
    # one good rock at Manhattan distance d from (0,3): 10 g^d + 10 g^6
    for j, d in ((1, 2), (3, 6), (6, 7), (7, 4), (0, 5)):
        assert m.upper(rs_state(7, 1 << j, [(0, 3)])) == pytest.approx(10 * g**d + 10 * g**6, rel=1e-14)
    # all eight good: distances 5 2 5 6 3 4 7 4 from (0,3)
    tot = sum(10 * g**d for d in (5, 2, 5, 6, 3, 4, 7, 4)) + 10 * g**6
    assert m.upper(rs_state(7, 0xFF, [(0, 3)])) == pytest.approx(tot, rel=1e-14)
    # on rock 5 (3,4), only it good: 10 + 10 g^3
    assert m.upper(rs_state(7, 1 << 5, [(3, 4)])) == pytest.approx(10 + 10 * g**3, rel=1e-14)
    # nothing good, robot at x = 2: 10 g^4
    assert m.upper(rs_state(7, 0, [(2, 5)])) == pytest.approx(10 * g**4, rel=1e-14)
    # exited: terminal, 0
    assert m.upper(rs_state(7, 0xFF, [None])) == 0.0


def test_mars_upper_bound_nearer_robot_and_exited_robot():
    params = "n=5 robots=2 D=20 gamma=0.95 rocks=2:1,1:4,3:0,3:3 starts=0:1,0:3"
    m = oracle.Model("rocksample", params)
    g = GAMMA
    # rock 3 (3,3) good; robot 0 at (0,1) (distance 5), robot 1 at (2,4) (distance 2)
    s = rs_state(5, 1 << 3, [(0, 1), (2, 4)])
    assert m.upper(s) == pytest.approx(10 * g**2 + 10 * g**4 + 10 * g**2, rel=1e-14)
    # robot 1 exited: robot 0's distance counts, one exit term
    s = rs_state(5, 1 << 3, [(0, 1), None])
    assert m.upper(s) == pytest.approx(10 * g**5 + 10 * g**4, rel=1e-14)
    # rocks 0 and 2 good, robots at (2,1) and (4,4): 10 + 10 g^2 (rock 2 from robot 0) + 10 g^2 + 10 g^0
    s = rs_state(5, 0b101, [(2, 1), (4, 4)])
    assert m.upper(s) == pytest.approx(10 + 10 * g**2 + 10 * g**2 + 10, rel=1e-14)


# ----------------------------------------------------------------------------
# Navigation pi0 (card: the first of [S, SE, SW, t even ? E : W, t even ? W : E]
# read FREE, else STAY).  Directions 1..8 = N NE E SE S SW W NW; observation
# bit k = direction k + 1, 1 = OCCUPIED.
# ----------------------------------------------------------------------------
N_, NE, E, SE, S, SW, W, NW = 1, 2, 3, 4, 5, 6, 7, 8


def occ(*dirs):
    z = 0
    for d in dirs:
        z |= 1 << (d - 1)
    return z


NAV_POLICY_CASES = [
    # (blocked directions, depth t, expected action)
    ((), 0, S), ((), 1, S),
    ((N_, NE, NW, E, W), 2, S),            # only S matters while S is free
    ((S,), 4, SE), ((S,), 5, SE),
    ((S, SE), 6, SW), ((S, SE), 7, SW),
    ((S, SE, SW), 8, E), ((S, SE, SW), 9, W),   # parity picks E (even) / W (odd)
    ((S, SE, SW, E), 10, W), ((S, SE, SW, W), 11, E),
    ((S, SE, SW, W), 12, E), ((S, SE, SW, E), 13, W),
    ((S, SE, SW, E, W), 14, 0), ((S, SE, SW, E, W), 15, 0),  # all five blocked: STAY
    ((S, SE, SW, E, W, N_, NE, NW), 3, 0),
    ((SE, SW, E, W), 1, S), ((S, SW, E, W), 0, SE),
]


@pytest.mark.parametrize("blocked,t,want", NAV_POLICY_CASES)
def test_nav_policy_every_branch(blocked, t, want):
    m = oracle.Model("nav", inputs.nav_params())
    s = np.zeros(m.SW, np.uint32)
    assert m.default_action(s, occ(*blocked), 0, t) == want


def test_nav_policy_ignores_north_readings():
    m = oracle.Model("nav", inputs.nav_params())
    s = np.zeros(m.SW, np.uint32)
    for t in (0, 1):
        for zn in range(8):  # every combination of N, NE, NW
            z = (zn & 1) << (N_ - 1) | ((zn >> 1) & 1) << (NE - 1) | ((zn >> 2) & 1) << (NW - 1)
            assert m.default_action(s, z | occ(S), 0, t) == SE


# ----------------------------------------------------------------------------
# Navigation u(s) = 20 g^(d-1): d = shortest 8-connected path to the goal on
# the obstacle-free grid whose wall row is closed except at the open gate
# (brute force BFS, every cell, both gates)
# ----------------------------------------------------------------------------
def bfs_from_goal(n, wall_y, gate_x, goal):
    dist = {goal: 0}
    q = deque([goal])
    while q:
        x, y = q.popleft()
        for dx in (-1, 0, 1):
            for dy in (-1, 0, 1):
                nx, ny = x + dx, y + dy
                if (dx, dy) == (0, 0) or not (0 <= nx < n and 0 <= ny < n) or (nx, ny) in dist:
                    continue
                if ny == wall_y and nx != gate_x:
                    continue
                dist[(nx, ny)] = dist[(x, y)] + 1
                q.append((nx, ny))
    return dist


@pytest.mark.parametrize("n,wall_y,gates,goal", [(13, 6, (3, 9), (6, 12)), (5, 2, (1, 3), (2, 4))])
def test_nav_upper_bound_equals_bfs_distance(n, wall_y, gates, goal):
    params = inputs.nav_params(n, wall_y=wall_y, gates=gates, goal=goal, landmarks=[] if n != 13 else None)
    m = oracle.Model("nav", params)
    checked = 0
    for g in (0, 1):
        dist = bfs_from_goal(n, wall_y, gates[g], goal)
        for (x, y), d in dist.items():
            if (x, y) == goal:
                continue
            s = np.zeros(m.SW, np.uint32)
            s[0] = (y * n + x) | (g << 8)
            assert m.upper(s) == pytest.approx(20 * GAMMA ** (d - 1), rel=1e-14), (x, y, g, d)
            checked += 1
    assert checked == 2 * (n * n - n)  # per gate: every cell off the wall row, plus the gate, minus the goal


# ----------------------------------------------------------------------------
# Driving heading noise ("Gaussian noises on their heading
# directions"; card sigma = pi/8)
# ----------------------------------------------------------------------------
GOALS = [(0.0, -10.0), (0.0, 10.0), (20.0, -10.0), (20.0, 10.0)]


def test_car_heading_noise_mean_zero_sigma_pi_over_8():
    m = oracle.Model("car", inputs.car_params(20))
    st = inputs.car_belief(1, 1004, 20)[:, 0]
    f = lambda w: float(np.uint32(w).view(np.float32))  # noqa: E731
    goals = [int((st[2 + i // 16] >> (2 * (i % 16))) & 3) for i in range(20)]
    angles = []
    for sid in range(5000):
        s2, _, _, _, _ = m.step(st, 0, sid, 1, 99)
        for i in range(20):
            x, y = f(st[4 + 2 * i]), f(st[5 + 2 * i])
            gx, gy = GOALS[goals[i]]
            ux, uy = gx - x, gy - y
            hx, hy = f(s2[4 + 2 * i]) - x, f(s2[5 + 2 * i]) - y
            angles.append(math.atan2(ux * hy - uy * hx, ux * hx + uy * hy))
    a = np.array(angles)
    assert a.size == 100000
    sd = a.std()
    assert abs(a.mean()) < 4 * sd / math.sqrt(a.size)  # mean 0
    assert abs(sd / (math.pi / 8) - 1) < 0.02, sd  # sigma = pi/8 within 2 %
    assert abs((a**3).mean()) / sd**3 < 0.03  # symmetric
    assert np.abs(a).max() < 3.2 * sd  # bounded (the four-byte sum is bounded)
    frac1 = (np.abs(a) < sd).mean()
    assert 0.64 < frac1 < 0.70, frac1  # bell-shaped: about 2/3 within one sigma
