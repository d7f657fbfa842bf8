"""ctypes wrapper of the CPU oracle (oracle/oracle.c).

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this package.  The product
path (paper_1802_06215_b200) never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "liboracle.so")
SRC = [os.path.join(HERE, "oracle.c"), os.path.join(HERE, "oracle.h")]
CFLAGS = ["-O2", "-std=c11", "-Wall", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared"]


def build(force=False):
    """Compile liboracle.so with plain IEEE fp (no contraction, no fast-math)."""
    if not force and os.path.exists(LIB) and all(os.path.getmtime(LIB) >= os.path.getmtime(s) for s in SRC):
        return LIB
    tmp = LIB + f".tmp{os.getpid()}"
    subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, SRC[0], "-lm"])
    os.replace(tmp, LIB)
    return LIB


class ModelInfo(C.Structure):
    _fields_ = [("num_actions", C.c_uint32), ("state_words", C.c_uint32), ("obs_words", C.c_uint32),
                ("obs_slots", C.c_uint32), ("max_depth", C.c_uint32), ("elements", C.c_uint32),
                ("gamma", C.c_double), ("tail", C.c_double)]


class Leaf(C.Structure):
    _fields_ = [("parent", C.c_int64), ("action", C.c_int32), ("child", C.c_uint32),
                ("depth", C.c_uint32), ("pad", C.c_uint32)]


class Expansion(C.Structure):
    _fields_ = [("node", C.c_void_p), ("n_scen", C.c_void_p), ("weight", C.c_void_p),
                ("act_reward", C.c_void_p), ("act_upper", C.c_void_p), ("act_lower", C.c_void_p),
                ("child_begin", C.c_void_p), ("child_capacity", C.c_uint32),
                ("child_count", C.c_void_p), ("child_first", C.c_void_p), ("child_weight", C.c_void_p),
                ("child_upper", C.c_void_p), ("child_lower", C.c_void_p), ("child_obs", C.c_void_p),
                ("scen_capacity", C.c_uint64), ("scen_obs", C.c_void_p), ("scen_reward", C.c_void_p),
                ("scen_upper", C.c_void_p), ("scen_lower", C.c_void_p), ("scen_len", C.c_void_p),
                ("scen_hash", C.c_void_p), ("scen_child", C.c_void_p), ("scen_states", C.c_void_p),
                ("scenario_steps", C.c_uint64)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(LIB)
        u32p, f32p, f64p = C.POINTER(C.c_uint32), C.POINTER(C.c_float), C.POINTER(C.c_double)
        L.oracle_philox4x32_10.argtypes = [u32p, u32p, u32p]
        L.oracle_threshold.argtypes = [C.c_double]
        L.oracle_threshold.restype = C.c_uint64
        L.oracle_model_load.argtypes = [C.c_char_p, C.c_char_p, C.POINTER(C.c_void_p)]
        L.oracle_model_free.argtypes = [C.c_void_p]
        L.oracle_model_info_get.argtypes = [C.c_void_p, C.POINTER(ModelInfo)]
        L.oracle_last_error.restype = C.c_char_p
        L.oracle_step.argtypes = [C.c_void_p, u32p, C.c_int32, C.c_uint32, C.c_uint32, C.c_uint64,
                                  u32p, u32p, f32p, C.POINTER(C.c_int32)]
        L.oracle_upper.argtypes = [C.c_void_p, u32p]
        L.oracle_upper.restype = C.c_double
        L.oracle_rollout.argtypes = [C.c_void_p, u32p, u32p, C.c_uint32, C.c_uint32, C.c_uint64,
                                     f64p, u32p, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
        L.oracle_default_action.argtypes = [C.c_void_p, u32p, u32p, C.c_uint64, C.c_uint32]
        L.oracle_default_action.restype = C.c_int32
        L.oracle_belief_load.argtypes = [C.c_void_p, u32p, f32p, C.c_uint32, C.c_uint64]
        L.oracle_belief_load.restype = C.c_int64
        L.oracle_node_size.argtypes = [C.c_void_p, C.c_int64, u32p, u32p]
        L.oracle_node_read.argtypes = [C.c_void_p, C.c_int64, u32p, f32p, u32p]
        L.oracle_node_release.argtypes = [C.c_void_p, C.c_int64]
        L.oracle_expand_batch.argtypes = [C.c_void_p, C.POINTER(Leaf), C.c_uint32, C.c_void_p,
                                          C.POINTER(Expansion)]
        L.oracle_rollout_bounds.argtypes = [C.c_void_p, C.c_int64, f64p, f64p, C.c_void_p, C.c_void_p]
        L.oracle_brute_force.argtypes = [C.c_void_p, C.c_int64, f64p]
        L.oracle_brute_force_q.argtypes = [C.c_void_p, C.c_int64, f64p]
        _lib = L
    return _lib


def _p(a, t):
    return a.ctypes.data_as(C.POINTER(t))


def philox(ctr, key):
    c = np.asarray(ctr, dtype=np.uint32)
    k = np.asarray(key, dtype=np.uint32)
    o = np.zeros(4, dtype=np.uint32)
    lib().oracle_philox4x32_10(_p(c, C.c_uint32), _p(k, C.c_uint32), _p(o, C.c_uint32))
    return o


def threshold(p):
    return int(lib().oracle_threshold(p))


class OracleError(RuntimeError):
    pass


def _check(rc):
    if rc < 0:
        raise OracleError(f"oracle error {rc}: {lib().oracle_last_error().decode()}")
    return rc


class Model:
    """One loaded model (an oracle_model*) plus its nodes."""

    def __init__(self, kind: str, params: str = ""):
        self.h = C.c_void_p()
        _check(lib().oracle_model_load(kind.encode(), params.encode(), C.byref(self.h)))
        info = ModelInfo()
        _check(lib().oracle_model_info_get(self.h, C.byref(info)))
        self.kind = kind
        self.params = params
        self.A = info.num_actions
        self.SW = info.state_words
        self.OW = info.obs_words
        self.slots = info.obs_slots
        self.D = info.max_depth
        self.elements = info.elements
        self.gamma = info.gamma
        self.tail = info.tail

    def __del__(self):
        try:
            if self.h:
                lib().oracle_model_free(self.h)
                self.h = C.c_void_p()
        except Exception:
            pass

    # ---- single-scenario primitives (pins) ----
    def step(self, s, a, sid, t, seed):
        s = np.ascontiguousarray(s, dtype=np.uint32)
        s2 = np.zeros(self.SW, np.uint32)
        z = np.zeros(self.OW, np.uint32)
        r = C.c_float()
        term = C.c_int32()
        counted = _check(lib().oracle_step(self.h, _p(s, C.c_uint32), int(a), int(sid), int(t), int(seed),
                                           _p(s2, C.c_uint32), _p(z, C.c_uint32), C.byref(r), C.byref(term)))
        return s2, z, float(r.value), bool(term.value), bool(counted)

    def upper(self, s):
        s = np.ascontiguousarray(s, dtype=np.uint32)
        return float(lib().oracle_upper(self.h, _p(s, C.c_uint32)))

    def rollout(self, s, z, sid, depth, seed):
        s = np.ascontiguousarray(s, dtype=np.uint32)
        zp = None
        if z is not None:
            z = np.ascontiguousarray(np.atleast_1d(z), dtype=np.uint32)
            zp = _p(z, C.c_uint32)
        ret = C.c_double()
        ln = C.c_uint32()
        h = C.c_uint64()
        st = C.c_uint64()
        _check(lib().oracle_rollout(self.h, _p(s, C.c_uint32), zp, int(sid), int(depth), int(seed),
                                    C.byref(ret), C.byref(ln), C.byref(h), C.byref(st)))
        return float(ret.value), int(ln.value), int(h.value), int(st.value)

    def default_action(self, s, z, memory, t):
        s = np.ascontiguousarray(s, dtype=np.uint32)
        z = np.ascontiguousarray(np.atleast_1d(z), dtype=np.uint32)
        return int(lib().oracle_default_action(self.h, _p(s, C.c_uint32), _p(z, C.c_uint32), int(memory), int(t)))

    # ---- nodes ----
    def belief_load(self, states_soa, weights, seed):
        st = np.ascontiguousarray(states_soa, dtype=np.uint32)
        w = np.ascontiguousarray(weights, dtype=np.float32)
        K = w.shape[0]
        assert st.shape == (self.SW, K), (st.shape, self.SW, K)
        h = lib().oracle_belief_load(self.h, _p(st, C.c_uint32), _p(w, C.c_float), K, int(seed))
        _check(h)
        return int(h)

    def node_read(self, node):
        n = C.c_uint32()
        d = C.c_uint32()
        _check(lib().oracle_node_size(self.h, node, C.byref(n), C.byref(d)))
        n = n.value
        ids = np.zeros(n, np.uint32)
        w = np.zeros(n, np.float32)
        st = np.zeros((self.SW, n), np.uint32)
        _check(lib().oracle_node_read(self.h, node, _p(ids, C.c_uint32), _p(w, C.c_float), _p(st, C.c_uint32)))
        return dict(ids=ids, w=w, states=st, depth=d.value)

    def node_release(self, node):
        _check(lib().oracle_node_release(self.h, node))

    def expand(self, leaves, action_mask=None, record=False, child_capacity=None):
        """leaves: list of (parent_node, action, child, depth).  Returns a dict
        of numpy arrays (fp64 values) mirroring despot_expansion."""
        Lc = len(leaves)
        A = self.A
        lv = (Leaf * Lc)()
        cap_s = 0
        for i, (p, a, c, d) in enumerate(leaves):
            lv[i].parent, lv[i].action, lv[i].child, lv[i].depth = int(p), int(a), int(c), int(d)
            n = C.c_uint32()
            _check(lib().oracle_node_size(self.h, int(p), C.byref(n), None))
            cap_s += n.value * A
        per_child = self.slots if self.slots else 1 << 30
        if child_capacity is None:
            child_capacity = 0
            for (p, a, c, d) in leaves:
                n = C.c_uint32()
                lib().oracle_node_size(self.h, int(p), C.byref(n), None)
                child_capacity += A * min(n.value, per_child)
        o = dict(
            node=np.zeros(Lc, np.int64), n_scen=np.zeros(Lc, np.uint32), weight=np.zeros(Lc),
            act_reward=np.zeros(Lc * A), act_upper=np.zeros(Lc * A), act_lower=np.zeros(Lc * A),
            child_begin=np.zeros(Lc * A + 1, np.uint32), child_count=np.zeros(child_capacity, np.uint32),
            child_first=np.zeros(child_capacity, np.uint32), child_weight=np.zeros(child_capacity),
            child_upper=np.zeros(child_capacity), child_lower=np.zeros(child_capacity),
            child_obs=np.zeros(child_capacity * self.OW, np.uint32))
        E = Expansion()
        for k in ("node", "n_scen", "weight", "act_reward", "act_upper", "act_lower", "child_begin",
                  "child_count", "child_first", "child_weight", "child_upper", "child_lower", "child_obs"):
            setattr(E, k, o[k].ctypes.data)
        E.child_capacity = child_capacity
        if record:
            S = cap_s
            o.update(scen_obs=np.zeros(S * self.OW, np.uint32), scen_reward=np.zeros(S, np.float32),
                     scen_upper=np.zeros(S), scen_lower=np.zeros(S), scen_len=np.zeros(S, np.uint32),
                     scen_hash=np.zeros(S, np.uint64), scen_child=np.zeros(S, np.uint32),
                     scen_states=np.zeros(S * self.SW, np.uint32))
            for k in ("scen_obs", "scen_reward", "scen_upper", "scen_lower", "scen_len", "scen_hash",
                      "scen_child", "scen_states"):
                setattr(E, k, o[k].ctypes.data)
            E.scen_capacity = S
        mask = None
        if action_mask is not None:
            mask = np.ascontiguousarray(action_mask, dtype=np.uint8)
        _check(lib().oracle_expand_batch(self.h, lv, Lc, mask.ctypes.data if mask is not None else None,
                                         C.byref(E)))
        C_tot = int(o["child_begin"][-1])
        for k in ("child_count", "child_first", "child_weight", "child_upper", "child_lower"):
            o[k] = o[k][:C_tot]
        o["child_obs"] = o["child_obs"][: C_tot * self.OW].reshape(C_tot, self.OW)
        if record:
            S = int(sum(int(n) for n in o["n_scen"]) * A)
            for k in ("scen_reward", "scen_upper", "scen_lower", "scen_len", "scen_hash", "scen_child"):
                o[k] = o[k][:S]
            o["scen_obs"] = o["scen_obs"][: S * self.OW].reshape(S, self.OW)
            o["scen_states"] = o["scen_states"][: S * self.SW].reshape(S, self.SW)
        o["scenario_steps"] = int(E.scenario_steps)
        return o

    def rollout_bounds(self, node, per_scenario=False):
        u = C.c_double()
        l = C.c_double()
        n = C.c_uint32()
        _check(lib().oracle_node_size(self.h, node, C.byref(n), None))
        pu = np.zeros(n.value)
        pl = np.zeros(n.value)
        _check(lib().oracle_rollout_bounds(self.h, node, C.byref(u), C.byref(l), pu.ctypes.data, pl.ctypes.data))
        if per_scenario:
            return u.value, l.value, pu, pl
        return u.value, l.value

    def brute_force(self, node):
        v = C.c_double()
        _check(lib().oracle_brute_force(self.h, node, C.byref(v)))
        return v.value

    def brute_force_q(self, node):
        q = np.zeros(self.A)
        _check(lib().oracle_brute_force_q(self.h, node, _p(q, C.c_double)))
        return q
