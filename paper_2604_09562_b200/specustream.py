"""ctypes binding of the SpecuStream depth controller in libsv.so (include/sv.h, NEXT-1;
PAPER.md Alg. 4). Argument marshalling only: the controller arithmetic runs in
csrc/specustream.cpp."""
import ctypes

from .sv import LaneStats, _check, load

SV_SPEC_MAX_H = 64


class SpecConfig(ctypes.Structure):
    _fields_ = [("d_base", ctypes.c_double), ("gamma", ctypes.c_double), ("d_min", ctypes.c_double),
                ("d_max", ctypes.c_double), ("h", ctypes.c_int32), ("projection_source", ctypes.c_int32),
                ("tau_target", ctypes.c_double), ("micro_batch_numerator", ctypes.c_double)]

    @classmethod
    def default(cls, **overrides):
        c = cls()
        _lib().sv_spec_default_config(ctypes.byref(c))
        for k, v in overrides.items():
            setattr(c, k, v)
        return c


class FlowState(ctypes.Structure):
    _fields_ = [("f", ctypes.c_double * SV_SPEC_MAX_H), ("idx", ctypes.c_int32), ("_pad", ctypes.c_int32),
                ("tau_recent", ctypes.c_double)]


class SpecPlan(ctypes.Structure):
    _fields_ = [("depth", ctypes.c_int32), ("micro_batch", ctypes.c_int32), ("projected", ctypes.c_double),
                ("raw_depth", ctypes.c_double), ("delta", ctypes.c_double), ("mag", ctypes.c_double),
                ("scale", ctypes.c_double), ("adj", ctypes.c_double)]

    def as_dict(self):
        return {n: getattr(self, n) for n, _ in self._fields_}


_sigs_done = False


def _lib():
    global _sigs_done
    lib = load()
    if not _sigs_done:
        P = ctypes.POINTER
        d = ctypes.c_double
        lib.sv_spec_default_config.argtypes, lib.sv_spec_default_config.restype = [P(SpecConfig)], None
        lib.sv_spec_reset.argtypes, lib.sv_spec_reset.restype = [P(SpecConfig), P(FlowState)], ctypes.c_int
        lib.sv_spec_adapt.argtypes = [P(SpecConfig), P(FlowState), d, d, d, P(SpecPlan), P(FlowState)]
        lib.sv_spec_adapt.restype = ctypes.c_int
        lib.sv_spec_step.argtypes = [P(SpecConfig), P(FlowState), P(LaneStats), P(LaneStats), d, ctypes.c_int32,
                                     ctypes.c_int32, P(SpecPlan), P(FlowState)]
        lib.sv_spec_step.restype = ctypes.c_int
        _sigs_done = True
    return lib


class Controller:
    """One lane's controller state (value-in / value-out underneath)."""

    def __init__(self, cfg=None):
        self.cfg = cfg if cfg is not None else SpecConfig.default()
        self.state = FlowState()
        _check(_lib().sv_spec_reset(ctypes.byref(self.cfg), ctypes.byref(self.state)), "sv_spec_reset")

    def adapt(self, a, l, t):
        plan, out = SpecPlan(), FlowState()
        _check(_lib().sv_spec_adapt(ctypes.byref(self.cfg), ctypes.byref(self.state), a, l, t, ctypes.byref(plan),
                                    ctypes.byref(out)), "sv_spec_adapt")
        self.state = out
        return plan

    def step(self, stats0, stats1, seconds, active, max_batch):
        """stats0 / stats1: LaneStats snapshots (sv.Lane.stats_raw()) `seconds` apart."""
        plan, out = SpecPlan(), FlowState()
        _check(_lib().sv_spec_step(ctypes.byref(self.cfg), ctypes.byref(self.state), ctypes.byref(stats0),
                                   ctypes.byref(stats1), seconds, active, max_batch, ctypes.byref(plan),
                                   ctypes.byref(out)), "sv_spec_step")
        self.state = out
        return plan

    def flow(self):
        return [self.state.f[j] for j in range(self.cfg.h)]
