"""Thin ctypes binding of libdespot (include/despot.h).

Argument marshalling only: every step of the batched leaf expansion runs in
the library's sm_100a kernels.  There is no CPU fallback -- if libdespot.so is
missing or no CUDA device is usable, calls raise DespotError.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DESPOT_LIB", os.path.join(HERE, "libdespot.so"))  # override: A/B builds

DESPOT_X_DEVICE_OUTPUTS = 1
DESPOT_X_RECORD_SCENARIO = 2
DESPOT_X_TIMING = 4
DESPOT_X_TIMING_K2 = 8
DESPOT_X_INDEX_LISTS = 16
DESPOT_X_RESIDENT = 32
DESPOT_MF_UNFACTORED = 1
DESPOT_MF_FACTORED = 2
DESPOT_MF_GROUPED = 4
DESPOT_MF_PAIRED = 16  # a lane pair per scenario (driving)
DESPOT_MF_EXCHANGE = 8  # run the sharded exchange path on the communicator even at world 1 (tests)

STATUS = {0: "OK", -1: "EINVAL", -2: "EMODEL", -3: "ENOMEM", -4: "ECAPACITY", -5: "ECUDA",
          -6: "ENCCL", -7: "ESHUTDOWN", -8: "EHASH"}

# every function declared in include/despot.h (checked by the CPU tests)
EXPORTS = ["despot_last_error", "despot_abi_version", "despot_model_load", "despot_model_info_get",
           "despot_model_free", "despot_belief_load", "despot_node_info", "despot_node_read",
           "despot_node_release", "despot_node_release_many", "despot_expand_batch", "despot_expand_begin", "despot_batch_exchange",
           "despot_expand_end", "despot_batch_abort", "despot_rollout_bounds", "despot_stream_words",
           "despot_search", "despot_plan", "despot_philox_ceiling", "despot_expand_batch_bytes",
           "despot_comm_unique_id", "despot_comm_init", "despot_comm_destroy", "despot_comm_info",
           "despot_batch_prepare", "despot_batch_run", "despot_batch_prepared_free"]


def _tflag(timing):
    """timing=True: every phase (8 CUDA events); "k2": K2 only (2 events, the
    cheap form for timing loops); False: none."""
    return DESPOT_X_TIMING_K2 if timing == "k2" else DESPOT_X_TIMING if timing else 0


class DespotError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code


DEV_ALLOC_FN = C.CFUNCTYPE(C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p)
DEV_FREE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_void_p, C.c_void_p)


class Opts(C.Structure):
    _fields_ = [("device", C.c_int), ("rank", C.c_int), ("world", C.c_int), ("flags", C.c_uint32),
                ("comm", C.c_void_p), ("dev_alloc", DEV_ALLOC_FN), ("dev_free", DEV_FREE_FN),
                ("alloc_ctx", C.c_void_p)]


def torch_allocator(device: int):
    """despot_opts allocator hooks backed by torch's caching allocator (node
    arenas and batch scratch then share torch's pool): (alloc, free) ctypes
    callbacks, to be kept alive as long as the model."""
    import torch

    def alloc(nbytes, stream, ctx):
        try:
            return torch.cuda.caching_allocator_alloc(int(nbytes), device, int(stream or 0))
        except Exception:  # ENOMEM for the library
            return None

    def free(ptr, stream, ctx):
        torch.cuda.caching_allocator_delete(int(ptr))

    return DEV_ALLOC_FN(alloc), DEV_FREE_FN(free)


class ModelInfo(C.Structure):
    _fields_ = [("num_actions", C.c_uint32), ("state_words", C.c_uint32), ("obs_words", C.c_uint32),
                ("obs_slots", C.c_uint32), ("max_depth", C.c_uint32), ("elements", C.c_uint32),
                ("gamma", C.c_double), ("tail", C.c_double)]


class Leaf(C.Structure):
    _fields_ = [("parent", C.c_uint64), ("action", C.c_int32), ("child", C.c_uint32),
                ("depth", C.c_uint32), ("pad", C.c_uint32)]


class Expansion(C.Structure):
    _fields_ = [("flags", C.c_uint32), ("node", C.c_void_p), ("n_scen", C.c_void_p), ("weight", C.c_void_p),
                ("act_reward", C.c_void_p), ("act_upper", C.c_void_p), ("act_lower", C.c_void_p),
                ("child_begin", C.c_void_p), ("child_capacity", C.c_uint32),
                ("child_count", C.c_void_p), ("child_first", C.c_void_p), ("child_weight", C.c_void_p),
                ("child_upper", C.c_void_p), ("child_lower", C.c_void_p), ("child_obs", C.c_void_p),
                ("scen_capacity", C.c_uint64), ("scen_obs", C.c_void_p), ("scen_reward", C.c_void_p),
                ("scen_upper", C.c_void_p), ("scen_lower", C.c_void_p), ("scen_len", C.c_void_p),
                ("scen_hash", C.c_void_p), ("scen_states", C.c_void_p),
                ("scenario_steps", C.c_uint64), ("num_children", C.c_uint32), ("launches", C.c_uint32),
                ("phase_ms", C.c_float * 4), ("h2d_bytes", C.c_uint64), ("d2h_bytes", C.c_uint64),
                ("exchange_ms", C.c_float), ("exchange_rounds", C.c_uint32), ("exchange_bytes", C.c_uint64),
                ("scen_child", C.c_void_p), ("index_begin", C.c_void_p), ("index", C.c_void_p)]


class SearchProblem(C.Structure):
    _fields_ = [("num_actions", C.c_uint32), ("obs_words", C.c_uint32), ("obs_slots", C.c_uint32),
                ("max_depth", C.c_uint32), ("gamma", C.c_double), ("root", C.c_uint64),
                ("root_depth", C.c_uint32), ("root_scenarios", C.c_uint32), ("root_weight", C.c_double),
                ("root_upper", C.c_double), ("root_lower", C.c_double), ("expand", C.c_void_p),
                ("release", C.c_void_p), ("ctx", C.c_void_p)]


class SearchConfig(C.Structure):
    _fields_ = [("workers", C.c_uint32), ("max_batch", C.c_uint32), ("max_inflight", C.c_uint32),
                ("batch_wait_us", C.c_uint32), ("max_trials", C.c_uint64), ("time_budget_s", C.c_double),
                ("xi", C.c_double), ("c_a", C.c_double), ("c_o", C.c_double), ("target_gap", C.c_double)]


class SearchResult(C.Structure):
    _fields_ = [("action", C.c_int32), ("root_upper", C.c_float), ("root_lower", C.c_float),
                ("nodes", C.c_uint64), ("expanded", C.c_uint64), ("trials", C.c_uint64), ("batches", C.c_uint64),
                ("max_depth", C.c_uint32), ("pad", C.c_uint32), ("seconds", C.c_double),
                ("scenario_steps", C.c_uint64)]


class SearchNode(C.Structure):
    _fields_ = [("parent", C.c_int32), ("action", C.c_int32), ("child", C.c_uint32), ("depth", C.c_uint32),
                ("n_scen", C.c_uint32), ("visits", C.c_uint32), ("branch_visits", C.c_uint32),
                ("active", C.c_int32), ("expanded", C.c_int32), ("weight", C.c_float), ("upper", C.c_float),
                ("lower", C.c_float), ("upper0", C.c_float), ("lower0", C.c_float)]


EXPAND_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_uint32, C.c_void_p)
RELEASE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_uint64)


def search_config(workers=1, max_batch=64, max_inflight=1, batch_wait_us=200, max_trials=0, time_budget_s=0.0,
                  xi=0.95, c_a=0.0, c_o=0.0, target_gap=0.0):
    return SearchConfig(workers, max_batch, max_inflight, batch_wait_us, max_trials, time_budget_s, xi, c_a, c_o,
                        target_gap)


def result_dict(r: SearchResult):
    return {k: getattr(r, k) for k, _ in SearchResult._fields_ if k != "pad"}


def search(problem: SearchProblem, config: SearchConfig, dump_capacity=0):
    """despot_search with a caller-provided backend (problem.expand/release
    hold CFUNCTYPE pointers the caller keeps alive)."""
    res = SearchResult()
    dump = (SearchNode * dump_capacity)() if dump_capacity else None
    _check(lib().despot_search(C.byref(problem), C.byref(config), C.byref(res), dump, dump_capacity))
    return result_dict(res), (list(dump)[: min(res.nodes, dump_capacity)] if dump_capacity else None)


class Exchange(C.Structure):
    _fields_ = [("sums", C.c_void_p), ("n_sums", C.c_uint64), ("mins", C.c_void_p), ("n_mins", C.c_uint64),
                ("maxs", C.c_void_p), ("n_maxs", C.c_uint64), ("gather", C.c_void_p), ("gather_bytes", C.c_uint64),
                ("round", C.c_uint32), ("more", C.c_uint32)]


_lib = None


def lib():
    """Load libdespot.so (in-tree).  Raises if it was not built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise DespotError(-5, f"{LIB_PATH} not built (run __graft_entry__.build())")
        L = C.CDLL(LIB_PATH)
        vp, u32, u64 = C.c_void_p, C.c_uint32, C.c_uint64
        L.despot_last_error.restype = C.c_char_p
        L.despot_model_load.argtypes = [C.c_char_p, C.c_char_p, C.POINTER(Opts), C.POINTER(vp)]
        L.despot_model_info_get.argtypes = [vp, C.POINTER(ModelInfo)]
        L.despot_model_free.argtypes = [vp]
        L.despot_belief_load.argtypes = [vp, vp, vp, u32, u64, vp, C.POINTER(u64)]
        L.despot_node_info.argtypes = [vp, u64, C.POINTER(u32), C.POINTER(u32)]
        L.despot_node_read.argtypes = [vp, u64, vp, vp, vp, vp]
        L.despot_node_release.argtypes = [vp, u64]
        L.despot_node_release_many.argtypes = [vp, C.POINTER(C.c_uint64), C.c_uint32]
        L.despot_expand_batch.argtypes = [vp, C.POINTER(Leaf), u32, C.POINTER(Expansion), vp]
        L.despot_expand_begin.argtypes = [vp, C.POINTER(Leaf), u32, u32, vp, C.POINTER(vp)]
        L.despot_batch_exchange.argtypes = [vp, C.POINTER(Exchange)]
        L.despot_expand_end.argtypes = [vp, C.POINTER(Expansion), vp]
        L.despot_batch_abort.argtypes = [vp]
        L.despot_rollout_bounds.argtypes = [vp, u64, C.POINTER(C.c_float), C.POINTER(C.c_float), vp, vp, vp]
        L.despot_stream_words.argtypes = [vp, u64, vp, u32, u32, u32, vp, vp]
        L.despot_expand_batch_bytes.argtypes = [vp, C.POINTER(Leaf), u32, u32, C.POINTER(C.c_uint32),
                                                C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
        L.despot_philox_ceiling.argtypes = [vp, u64, u32, u32, u32, vp, C.POINTER(C.c_double),
                                            C.POINTER(C.c_uint32)]
        L.despot_search.argtypes = [C.POINTER(SearchProblem), C.POINTER(SearchConfig), C.POINTER(SearchResult),
                                    vp, u32]
        L.despot_plan.argtypes = [vp, u64, C.POINTER(SearchConfig), C.POINTER(SearchResult), vp]
        L.despot_batch_prepare.argtypes = [vp, C.POINTER(Leaf), u32, C.POINTER(Expansion), C.POINTER(vp)]
        L.despot_batch_run.argtypes = [vp, C.POINTER(Expansion), vp]
        L.despot_batch_prepared_free.argtypes = [vp]
        L.despot_comm_unique_id.argtypes = [vp]
        L.despot_comm_init.argtypes = [vp, C.c_int, C.c_int, C.c_int, C.POINTER(vp)]
        L.despot_comm_destroy.argtypes = [vp]
        L.despot_comm_info.argtypes = [vp, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int)]
        _lib = L
    return _lib


def _check(rc):
    if rc != 0:
        raise DespotError(rc, lib().despot_last_error().decode())


def _stream_ptr(stream):
    if stream is None:
        try:
            import torch
            if torch.cuda.is_available():
                return torch.cuda.current_stream().cuda_stream
        except Exception:
            pass
        return None
    return getattr(stream, "cuda_stream", stream)


def comm_unique_id() -> bytes:
    """despot_comm_unique_id: the 128-byte NCCL unique id (rank 0 creates it,
    every rank receives it over the caller's channel)."""
    buf = C.create_string_buffer(128)
    _check(lib().despot_comm_unique_id(buf))
    return buf.raw


class Comm:
    """A communicator owned by the library (despot_comm_init): models loaded
    with it run sharded batches, their exchange included, in one call."""

    def __init__(self, uid: bytes, rank: int, world: int, device: int = 0):
        if len(uid) != 128:
            raise DespotError(-1, "the unique id is 128 bytes")
        self.h = C.c_void_p()
        buf = C.create_string_buffer(bytes(uid), 128)
        _check(lib().despot_comm_init(buf, int(rank), int(world), int(device), C.byref(self.h)))
        self.rank, self.world, self.device = rank, world, device

    def info(self):
        r, w, v = C.c_int(), C.c_int(), C.c_int()
        _check(lib().despot_comm_info(self.h, C.byref(r), C.byref(w), C.byref(v)))
        return {"rank": r.value, "world": w.value, "nccl_version": v.value}

    def close(self):
        if self.h:
            lib().despot_comm_destroy(self.h)
            self.h = C.c_void_p()


class _Prepared:
    """Owner of a despot_prepared: freed with the prepared dict, or by the
    model's close() (whichever comes first)."""

    def __init__(self, h, model):
        self.h = h
        model._prepared.add(self)

    def free(self):
        if self.h:
            lib().despot_batch_prepared_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class Model:
    """A loaded model (despot_model*)."""

    def __init__(self, kind: str, params: str = "", device: int = 0, rank: int = 0, world: int = 1,
                 flags: int = 0, comm: "Comm | None" = None, allocator: "str | None" = None):
        """allocator: None (the library's stream-ordered cudaMallocAsync) or
        "torch" (torch's caching allocator through despot_opts' hooks)."""
        self.h = C.c_void_p()
        self.comm = comm  # kept alive as long as the model
        import weakref
        self._prepared = weakref.WeakSet()
        self._hooks = torch_allocator(device) if allocator == "torch" else (DEV_ALLOC_FN(), DEV_FREE_FN())
        o = Opts(device, rank, world, flags, comm.h.value if comm is not None else None, self._hooks[0],
                 self._hooks[1], None)
        _check(lib().despot_model_load(kind.encode(), params.encode(), C.byref(o), C.byref(self.h)))
        info = ModelInfo()
        _check(lib().despot_model_info_get(self.h, C.byref(info)))
        self.kind, self.params, self.device, self.rank, self.world = kind, params, device, rank, world
        self.A, self.SW, self.OW = info.num_actions, info.state_words, info.obs_words
        self.slots, self.D, self.elements = info.obs_slots, info.max_depth, info.elements
        self.gamma, self.tail = info.gamma, info.tail

    def close(self):
        for p in list(self._prepared):
            p.free()
        if self.h:
            lib().despot_model_free(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- nodes ----
    def belief_load(self, states_soa, weights, seed, stream=None) -> int:
        st = np.ascontiguousarray(states_soa, dtype=np.uint32)
        w = np.ascontiguousarray(weights, dtype=np.float32)
        K = int(w.shape[0])
        if st.shape != (self.SW, K):
            raise DespotError(-1, f"states must be [{self.SW}][{K}]")
        out = C.c_uint64()
        _check(lib().despot_belief_load(self.h, st.ctypes.data, w.ctypes.data, K, int(seed),
                                        _stream_ptr(stream), C.byref(out)))
        return int(out.value)

    def node_info(self, node):
        n, d = C.c_uint32(), C.c_uint32()
        _check(lib().despot_node_info(self.h, int(node), C.byref(n), C.byref(d)))
        return int(n.value), int(d.value)

    def node_read(self, node, stream=None):
        n, d = self.node_info(node)
        ids = np.zeros(n, np.uint32)
        w = np.zeros(n, np.float32)
        st = np.zeros((self.SW, n), np.uint32)
        _check(lib().despot_node_read(self.h, int(node), ids.ctypes.data, w.ctypes.data, st.ctypes.data,
                                      _stream_ptr(stream)))
        return dict(ids=ids, w=w, states=st, depth=d)

    def node_release(self, node):
        _check(lib().despot_node_release(self.h, int(node)))

    def node_release_many(self, nodes):
        """Releases every node in `nodes` (one foreign call)."""
        arr = (C.c_uint64 * len(nodes))(*[int(n) for n in nodes])
        _check(lib().despot_node_release_many(self.h, arr, len(nodes)))

    # ---- expansion ----
    @staticmethod
    def _leaves(leaves):
        Lc = len(leaves)
        lv = (Leaf * Lc)()
        for i, (p, a, c, d) in enumerate(leaves):
            lv[i].parent, lv[i].action, lv[i].child, lv[i].depth = int(p), int(a), int(c), int(d)
        return lv

    def child_capacity_bound(self, leaves):
        """Children bound of a batch: A * min(|Phi|, slots) per leaf.  Under
        sharding |Phi| is global and only the local count is known here, so
        the bound is (n + 1) * world -- exact for interleaved roots; a
        filtered node may need more, which the call reports as ECAPACITY."""
        per = self.slots if self.slots else None
        W = max(self.world, 1)
        tot = 0
        for (p, a, c, d) in leaves:
            n, _ = self.node_info(p)
            g = n if W == 1 else (n + 1) * W
            tot += self.A * (min(g, per) if per else g)
        return max(tot, 1)

    def _alloc_outputs(self, L, C_cap, S_cap, record, device, pinned=False):
        A, OW, SW = self.A, self.OW, self.SW
        keep = []
        if pinned and not device:
            # page-locked host arrays (numpy views of pinned torch buffers): the
            # library copies the results straight into them
            import torch

            def z(n, dt):
                n = max(int(n), 1)
                t = torch.zeros(n * np.dtype(dt).itemsize, dtype=torch.uint8, pin_memory=True)
                keep.append(t)
                return t.numpy().view(dt)
            u32, f32, i64 = np.uint32, np.float32, np.uint64
            ptr = lambda t: t.ctypes.data  # noqa: E731
        elif device:
            import torch
            dev = torch.device("cuda", self.device)
            z = lambda n, dt: torch.zeros(max(int(n), 1), dtype=dt, device=dev)  # noqa: E731
            u32, f32, i64 = torch.int32, torch.float32, torch.int64
            ptr = lambda t: t.data_ptr()  # noqa: E731
        else:
            z = lambda n, dt: np.zeros(max(int(n), 1), dtype=dt)  # noqa: E731
            u32, f32, i64 = np.uint32, np.float32, np.uint64
            ptr = lambda t: t.ctypes.data  # noqa: E731
        o = dict(n_scen=z(L, u32), weight=z(L, f32), act_reward=z(L * A, f32), act_upper=z(L * A, f32),
                 act_lower=z(L * A, f32), child_begin=z(L * A + 1, u32), child_count=z(C_cap, u32),
                 child_first=z(C_cap, u32), child_weight=z(C_cap, f32), child_upper=z(C_cap, f32),
                 child_lower=z(C_cap, f32), child_obs=z(C_cap * OW, u32))
        if record:
            o.update(scen_obs=z(S_cap * OW, u32), scen_reward=z(S_cap, f32), scen_upper=z(S_cap, f32),
                     scen_lower=z(S_cap, f32), scen_len=z(S_cap, u32), scen_hash=z(S_cap, i64),
                     scen_states=z(S_cap * SW, u32), scen_child=z(S_cap, u32))
        E = Expansion()
        for k, v in o.items():
            setattr(E, k, ptr(v))
        if keep:
            o["_pinned"] = keep  # owners of the page-locked memory
        E.child_capacity = int(C_cap)
        E.scen_capacity = int(S_cap) if record else 0
        return o, E

    def _finish(self, o, E, L, nodes, record, device):
        A = self.A
        Cn = int(E.num_children)
        out = dict(o)
        out["node"] = [int(x) for x in nodes]
        out["scenario_steps"] = int(E.scenario_steps)
        out["num_children"] = Cn
        out["phase_ms"] = [float(x) for x in E.phase_ms]
        out["launches"] = int(E.launches)
        out["h2d_bytes"], out["d2h_bytes"] = int(E.h2d_bytes), int(E.d2h_bytes)
        out["exchange_ms"], out["exchange_rounds"] = float(E.exchange_ms), int(E.exchange_rounds)
        out["exchange_bytes"] = int(E.exchange_bytes)
        if not device:
            for k in ("child_count", "child_first", "child_weight", "child_upper", "child_lower"):
                out["_full_" + k] = o[k]  # the whole capacity (self-check runs: nothing written past Cn)
                out[k] = o[k][:Cn]
            out["child_obs"] = o["child_obs"][: Cn * self.OW].reshape(Cn, self.OW)
            if record:
                S = int(o["n_scen"].astype(np.int64).sum()) * A
                for k in ("scen_reward", "scen_upper", "scen_lower", "scen_len", "scen_hash", "scen_child"):
                    out[k] = o[k][:S]
                out["scen_obs"] = o["scen_obs"][: S * self.OW].reshape(S, self.OW)
                out["scen_states"] = o["scen_states"][: S * self.SW].reshape(S, self.SW)
        return out

    def expand(self, leaves, record=False, device_outputs=False, child_capacity=None, scen_capacity=None,
               stream=None, timing=False, outputs=None, index_lists=None):
        """leaves: list of (node, action, child, depth).  Returns a dict of
        arrays (numpy, or torch CUDA tensors with device_outputs=True).
        index_lists: per leaf, the parent positions it holds (the paper's
        update form, DESPOT_X_INDEX_LISTS; [] for self leaves)."""
        L = len(leaves)
        lv = self._leaves(leaves)
        C_cap = child_capacity
        if C_cap is None and outputs is None:
            C_cap = self.child_capacity_bound(leaves)
        S_cap = 0
        if record:
            S_cap = scen_capacity if scen_capacity is not None else sum(self.A * self.node_info(p)[0]
                                                                         for (p, a, c, d) in leaves)
        if outputs is None:
            o, E = self._alloc_outputs(L, C_cap, S_cap, record, device_outputs)
        else:  # reuse preallocated buffers (bench): (dict, Expansion)
            o, E = outputs
        nodes = (C.c_uint64 * L)()
        E.node = C.addressof(nodes)
        E.flags = ((DESPOT_X_DEVICE_OUTPUTS if device_outputs else 0) | (DESPOT_X_RECORD_SCENARIO if record else 0)
                   | _tflag(timing))
        keep_idx = None
        if index_lists is not None:
            begin = np.zeros(L + 1, np.uint32)
            begin[1:] = np.cumsum([len(x) for x in index_lists])
            idx = np.ascontiguousarray(np.concatenate([np.asarray(x, np.uint32) for x in index_lists])
                                       if int(begin[-1]) else np.zeros(1, np.uint32), dtype=np.uint32)
            keep_idx = (begin, idx)
            E.flags |= DESPOT_X_INDEX_LISTS
            E.index_begin, E.index = begin.ctypes.data, idx.ctypes.data
        _check(lib().despot_expand_batch(self.h, lv, L, C.byref(E), _stream_ptr(stream)))
        del keep_idx
        return self._finish(o, E, L, nodes, record, device_outputs)

    # ---- prepared calls (repeated batches: no per-call marshalling) ----
    def prepare(self, leaves, device_outputs=False, child_capacity=None, timing=False, pinned=False, graph=True,
                resident=False):
        """A repeated batch: the leaf table, output arrays and expansion struct
        built once, and (graph=True, single GPU) despot_batch_prepare's CUDA
        graph of the batch's device work; `run_prepared` then costs one
        foreign call (despot_batch_run: new arenas, leaf-table patch, one
        graph launch).  pinned: host outputs in page-locked memory (copied
        into directly).  resident: DESPOT_X_RESIDENT (self leaves, small
        batch: the graph is K2 alone)."""
        L = len(leaves)
        C_cap = child_capacity if child_capacity is not None else self.child_capacity_bound(leaves)
        o, E = self._alloc_outputs(L, C_cap, 0, False, device_outputs, pinned=pinned)
        nodes = (C.c_uint64 * L)()
        E.node = C.addressof(nodes)
        E.flags = ((DESPOT_X_DEVICE_OUTPUTS if device_outputs else 0) | _tflag(timing) |
                   (DESPOT_X_RESIDENT if resident else 0))
        prep = {"lv": self._leaves(leaves), "L": L, "E": E, "o": o, "nodes": nodes, "ref": C.byref(E),
                "leaves": list(leaves), "graph": None}
        if graph and self.world == 1 and self.comm is None:
            g = C.c_void_p()
            _check(lib().despot_batch_prepare(self.h, prep["lv"], L, prep["ref"], C.byref(g)))
            prep["graph"] = _Prepared(g, self)
        return prep

    def run_prepared(self, prep, stream=None):
        """One run of a prepared batch; returns (scenario_steps, launches,
        node handles); outputs are in prep["o"], prep["E"]."""
        if prep["graph"] is not None:
            _check(lib().despot_batch_run(prep["graph"].h, prep["ref"], _stream_ptr(stream)))
        else:
            _check(lib().despot_expand_batch(self.h, prep["lv"], prep["L"], prep["ref"], _stream_ptr(stream)))
        E = prep["E"]
        return E.scenario_steps, E.launches, prep["nodes"]

    # ---- two-phase form for scenario sharding ----
    def alloc_outputs(self, leaves, device_outputs=False, child_capacity=None, pinned=False):
        C_cap = child_capacity if child_capacity is not None else self.child_capacity_bound(leaves)
        return self._alloc_outputs(len(leaves), C_cap, 0, False, device_outputs, pinned=pinned)

    def expand_begin(self, leaves, record=False, stream=None, timing=False):
        lv = self._leaves(leaves)
        b = C.c_void_p()
        flags = (DESPOT_X_RECORD_SCENARIO if record else 0) | _tflag(timing)
        _check(lib().despot_expand_begin(self.h, lv, len(leaves), flags, _stream_ptr(stream), C.byref(b)))
        ex = Exchange()
        _check(lib().despot_batch_exchange(b, C.byref(ex)))
        return b, ex

    def expand_end(self, batch, leaves, device_outputs=False, child_capacity=None, stream=None, timing=False,
                   outputs=None):
        L = len(leaves)
        if outputs is None:
            C_cap = child_capacity if child_capacity is not None else self.child_capacity_bound(leaves)
            o, E = self._alloc_outputs(L, C_cap, 0, False, device_outputs)
        else:
            o, E = outputs
        nodes = (C.c_uint64 * L)()
        E.node = C.addressof(nodes)
        E.flags = (DESPOT_X_DEVICE_OUTPUTS if device_outputs else 0) | _tflag(timing)
        _check(lib().despot_expand_end(batch, C.byref(E), _stream_ptr(stream)))
        return self._finish(o, E, L, nodes, False, device_outputs)

    def batch_exchange(self, batch):
        """The next exchange round of a sharded batch (after the caller ran
        the previous round's collectives); see dist.run_exchange."""
        ex = Exchange()
        _check(lib().despot_batch_exchange(batch, C.byref(ex)))
        return ex

    def batch_abort(self, batch):
        _check(lib().despot_batch_abort(batch))

    def rollout_bounds(self, node, per_scenario=False, stream=None):
        n, _ = self.node_info(node)
        u, l = C.c_float(), C.c_float()
        pu = np.zeros(max(n, 1), np.float32)
        pl = np.zeros(max(n, 1), np.float32)
        _check(lib().despot_rollout_bounds(self.h, int(node), C.byref(u), C.byref(l), pu.ctypes.data,
                                           pl.ctypes.data, _stream_ptr(stream)))
        if per_scenario:
            return u.value, l.value, pu[:n], pl[:n]
        return u.value, l.value

    def plan(self, root, config=None, stream=None, **kw):
        """Parallel DESPOT search from `root` on the GPU backend (despot_plan)."""
        cfg = config if config is not None else search_config(**kw)
        res = SearchResult()
        _check(lib().despot_plan(self.h, int(root), C.byref(cfg), C.byref(res), _stream_ptr(stream)))
        return result_dict(res)

    def batch_bytes(self, leaves, record=False):
        """despot_expand_batch_bytes: (child_capacity, scen_capacity, host
        output bytes) of a batch."""
        c, sc, hb = C.c_uint32(), C.c_uint64(), C.c_uint64()
        _check(lib().despot_expand_batch_bytes(self.h, self._leaves(leaves), len(leaves),
                                               DESPOT_X_RECORD_SCENARIO if record else 0, C.byref(c),
                                               C.byref(sc), C.byref(hb)))
        return c.value, sc.value, hb.value

    def philox_ceiling(self, seed, n_threads, blocks, reps=5, stream=None):
        """K0 (despot_philox_ceiling): (ms per launch of n_threads * blocks
        Philox blocks, XOR checksum of one launch's words)."""
        ms, cs = C.c_double(), C.c_uint32()
        _check(lib().despot_philox_ceiling(self.h, int(seed), int(n_threads), int(blocks), int(reps),
                                           _stream_ptr(stream), C.byref(ms), C.byref(cs)))
        return ms.value, cs.value

    def stream_words(self, seed, ids, t, k, stream=None):
        ids = np.ascontiguousarray(ids, dtype=np.uint32)
        out = np.zeros(len(ids), np.uint32)
        _check(lib().despot_stream_words(self.h, int(seed), ids.ctypes.data, len(ids), int(t), int(k),
                                         out.ctypes.data, _stream_ptr(stream)))
        return out
