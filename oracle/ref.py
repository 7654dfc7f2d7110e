"""TEST INFRASTRUCTURE ONLY: ctypes binding to oracle/_ref/libdeltaref.so,
the unmodified reference simulator (see oracle/Makefile, oracle/ref_shim.cpp).
"""
from __future__ import annotations

import ctypes as C
import json
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libdeltaref.so")


class RefConfig(C.Structure):
    _fields_ = [
        ("budget", C.c_uint64), ("heuristic", C.c_uint32), ("policy", C.c_uint32),
        ("bw_num", C.c_uint64), ("bw_den", C.c_uint64), ("eff_num", C.c_uint64),
        ("eff_den", C.c_uint64), ("swap_mode", C.c_uint32), ("guard", C.c_uint32),
        ("wm_num", C.c_uint64), ("wm_den", C.c_uint64), ("prefetch_limit", C.c_uint64),
        ("prefetch_enabled", C.c_uint32), ("overlap_enabled", C.c_uint32),
        ("scripted_nodes", C.POINTER(C.c_uint64)), ("scripted_actions", C.POINTER(C.c_uint32)),
        ("n_scripted", C.c_uint64),
    ]


def available() -> bool:
    return os.path.exists(LIB_PATH)


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise FileNotFoundError(f"{LIB_PATH} not built (make -C oracle)")
        L = C.CDLL(LIB_PATH)
        vp = C.c_void_p
        for name, res, args in [
            ("dref_run", vp, [C.c_char_p, C.POINTER(RefConfig), C.c_int]),
            ("dref_report", vp, [C.c_char_p, C.POINTER(RefConfig)]),
            ("dref_time_run", C.c_double, [C.c_char_p, C.POINTER(RefConfig), C.c_int]),
            ("dref_replay_check", vp, [C.c_char_p, C.POINTER(RefConfig), C.c_char_p]),
            ("dref_brute_force", C.c_uint64, [C.c_char_p, C.c_uint64]),
            ("dref_generate", vp, [C.c_int, C.c_uint64, C.c_uint64]),
            ("dref_comparison", vp, [C.c_char_p, C.POINTER(RefConfig), C.POINTER(C.c_uint64),
                                     C.c_uint64, C.POINTER(C.c_uint32), C.c_uint64,
                                     C.POINTER(C.c_uint32), C.c_uint64, C.c_int]),
            ("dref_free", None, [vp]),
        ]:
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def config(budget: int, bandwidth_bytes_per_us=(64000, 1), effective_fraction=(7, 20),
           policy_mode: int = 0, heuristic: int = 0):
    """An EngineConfig-like object with the reference defaults
    (include/deltasim/engine.hpp:25-40, policy.hpp:18-26) — lets the
    reference arm drive the oracle without importing the product."""
    from types import SimpleNamespace
    cm = SimpleNamespace(bandwidth_bytes_per_us=tuple(bandwidth_bytes_per_us),
                         effective_fraction=tuple(effective_fraction), swap_cost_mode=0)
    return SimpleNamespace(budget=int(budget), heuristic=heuristic, policy_mode=policy_mode,
                           cost_model=cm, watermark_fraction=(3, 4), prefetch_limit=2,
                           prefetch_enabled=True, overlap_enabled=True, prefetch_guard=0,
                           scripted_decisions=[])


def _cfg(cfg) -> tuple:
    """Accepts a paper_2203_15980_b200.planner.EngineConfig-like object."""
    c = RefConfig()
    c.budget = cfg.budget
    c.heuristic = int(cfg.heuristic)
    c.policy = int(cfg.policy_mode)
    c.bw_num, c.bw_den = cfg.cost_model.bandwidth_bytes_per_us
    c.eff_num, c.eff_den = cfg.cost_model.effective_fraction
    c.swap_mode = int(cfg.cost_model.swap_cost_mode)
    c.guard = int(cfg.prefetch_guard)
    c.wm_num, c.wm_den = cfg.watermark_fraction
    c.prefetch_limit = cfg.prefetch_limit
    c.prefetch_enabled = int(bool(cfg.prefetch_enabled))
    c.overlap_enabled = int(bool(cfg.overlap_enabled))
    keep = []
    if cfg.scripted_decisions:
        n = len(cfg.scripted_decisions)
        nodes = (C.c_uint64 * n)(*[a for a, _ in cfg.scripted_decisions])
        acts = (C.c_uint32 * n)(*[int(b) for _, b in cfg.scripted_decisions])
        c.scripted_nodes = C.cast(nodes, C.POINTER(C.c_uint64))
        c.scripted_actions = C.cast(acts, C.POINTER(C.c_uint32))
        c.n_scripted = n
        keep = [nodes, acts]
    return c, keep


def _take(p) -> str:
    try:
        return C.string_at(p).decode()
    finally:
        lib().dref_free(p)


def run(trace_json: str, cfg, baseline: bool = False) -> dict:
    """run_iteration / run_unconstrained_baseline of the reference."""
    c, keep = _cfg(cfg)
    return json.loads(_take(lib().dref_run(trace_json.encode(), C.byref(c), int(baseline))))


def report(trace_json: str, cfg) -> str:
    c, keep = _cfg(cfg)
    return _take(lib().dref_report(trace_json.encode(), C.byref(c)))


def time_run_ns(trace_json: str, cfg, iters: int) -> float:
    c, keep = _cfg(cfg)
    return lib().dref_time_run(trace_json.encode(), C.byref(c), iters)


def replay_check(trace_json: str, cfg, chrome_json: str) -> list:
    c, keep = _cfg(cfg)
    out = json.loads(_take(lib().dref_replay_check(trace_json.encode(), C.byref(c),
                                                   chrome_json.encode())))
    if isinstance(out, dict):
        raise RuntimeError(out.get("what"))
    return out


def comparison(trace_json: str, cfg, budgets, policies, heuristics, fmt: str = "csv") -> str:
    """the reference's run_comparison rendered by comparison_to_csv / _json.
    Runs in a fresh interpreter: this entry point crashes when libdelta is
    mapped into the same process (a symbol-interposition clash not yet
    isolated; every other entry point is unaffected)."""
    import subprocess
    import sys
    payload = json.dumps({"trace": trace_json, "budgets": list(budgets),
                          "policies": [int(x) for x in policies],
                          "heuristics": [int(x) for x in heuristics], "fmt": fmt,
                          "cfg": {"budget": cfg.budget, "heuristic": int(cfg.heuristic),
                                  "policy_mode": int(cfg.policy_mode),
                                  "bw": list(cfg.cost_model.bandwidth_bytes_per_us),
                                  "eff": list(cfg.cost_model.effective_fraction),
                                  "swap": int(cfg.cost_model.swap_cost_mode),
                                  "wm": list(cfg.watermark_fraction),
                                  "limit": cfg.prefetch_limit, "pf": bool(cfg.prefetch_enabled),
                                  "ov": bool(cfg.overlap_enabled),
                                  "guard": int(cfg.prefetch_guard)}})
    code = ("import json, sys; sys.path.insert(0, %r); from oracle import ref; "
            "d = json.loads(sys.stdin.read()); sys.stdout.write(ref._comparison_inproc(d))"
            % os.path.dirname(HERE))
    out = subprocess.run([sys.executable, "-c", code], input=payload, capture_output=True,
                         text=True, check=True)
    return out.stdout


def _comparison_inproc(d: dict) -> str:
    from types import SimpleNamespace
    c_ = d["cfg"]
    cfg = config(c_["budget"], tuple(c_["bw"]), tuple(c_["eff"]), c_["policy_mode"], c_["heuristic"])
    cfg.cost_model.swap_cost_mode = c_["swap"]
    cfg.watermark_fraction = tuple(c_["wm"])
    cfg.prefetch_limit = c_["limit"]
    cfg.prefetch_enabled = c_["pf"]
    cfg.overlap_enabled = c_["ov"]
    cfg.prefetch_guard = c_["guard"]
    del SimpleNamespace
    trace_json, budgets, policies, heuristics = d["trace"], d["budgets"], d["policies"], d["heuristics"]
    fmt = d["fmt"]
    c, keep = _cfg(cfg)
    b = (C.c_uint64 * max(1, len(budgets)))(*budgets)
    p = (C.c_uint32 * max(1, len(policies)))(*[int(x) for x in policies])
    h = (C.c_uint32 * max(1, len(heuristics)))(*[int(x) for x in heuristics])
    return _take(lib().dref_comparison(trace_json.encode(), C.byref(c), b, len(budgets), p,
                                       len(policies), h, len(heuristics), int(fmt == "json")))


def brute_force(trace_json: str, max_nodes: int = 12) -> int:
    return lib().dref_brute_force(trace_json.encode(), max_nodes)


def generate(kind: str, n: int, seed: int = 0) -> str:
    k = {"linear": 0, "resnet": 1, "transformer": 2}[kind]
    return _take(lib().dref_generate(k, n, seed))
