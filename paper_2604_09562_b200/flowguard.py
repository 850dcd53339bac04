"""ctypes binding of the FlowGuard lane router in libsv.so (include/sv.h, NEXT-2; §3.3,
Alg. 2). Argument marshalling only: the routing arithmetic runs in csrc/flowguard.cpp."""
import ctypes
import math

from .sv import _check, load


class RouteConfig(ctypes.Structure):
    _fields_ = [("alpha", ctypes.c_double * 4), ("tau", ctypes.c_double), ("q_max", ctypes.c_double),
                ("staleness_ms", ctypes.c_int64)]

    @classmethod
    def default(cls, **overrides):
        c = cls()
        _lib().sv_route_default_config(ctypes.byref(c))
        for k, v in overrides.items():
            if k == "alpha":
                for j in range(4):
                    c.alpha[j] = v[j]
            else:
                setattr(c, k, v)
        return c


class LaneMetrics(ctypes.Structure):
    _fields_ = [("timestamp_ms", ctypes.c_int64), ("cache_hit", ctypes.c_double), ("mem_util", ctypes.c_double),
                ("queue_depth", ctypes.c_double), ("active_load", ctypes.c_double)]


SV_ROUTE_OVERLOADED, SV_ROUTE_STALE = 1, 2
_sigs = False


def _lib():
    global _sigs
    lib = load()
    if not _sigs:
        P = ctypes.POINTER
        lib.sv_route_default_config.argtypes, lib.sv_route_default_config.restype = [P(RouteConfig)], None
        lib.sv_route_select.argtypes = [P(RouteConfig), ctypes.c_int32, P(LaneMetrics), P(ctypes.c_double),
                                        ctypes.c_int64, P(ctypes.c_int32), P(ctypes.c_double), P(ctypes.c_uint8),
                                        P(ctypes.c_int32)]
        lib.sv_route_select.restype = ctypes.c_int
        _sigs = True
    return lib


def select(metrics, live_queue=None, now_ms=0, cfg=None):
    """metrics: list of dicts / tuples (timestamp_ms, cache_hit, mem_util, queue_depth, active_load).
    Returns (chosen, scores (None where excluded), flags, used_fallback)."""
    cfg = cfg if cfg is not None else RouteConfig.default()
    n = len(metrics)
    arr = (LaneMetrics * max(1, n))()
    for i, m in enumerate(metrics):
        vals = (m["timestamp_ms"], m["cache_hit"], m["mem_util"], m["queue_depth"], m["active_load"]) \
            if isinstance(m, dict) else tuple(m)
        arr[i] = LaneMetrics(*vals)
    live = None if live_queue is None else (ctypes.c_double * n)(*[float(x) for x in live_queue])
    chosen, fb = ctypes.c_int32(), ctypes.c_int32()
    scores, flags = (ctypes.c_double * max(1, n))(), (ctypes.c_uint8 * max(1, n))()
    _check(_lib().sv_route_select(ctypes.byref(cfg), n, arr, live, int(now_ms), ctypes.byref(chosen), scores, flags,
                                  ctypes.byref(fb)), "sv_route_select")
    sc = [None if math.isnan(scores[i]) else scores[i] for i in range(n)]
    return chosen.value, sc, [int(flags[i]) for i in range(n)], bool(fb.value)
