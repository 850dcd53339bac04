"""CPU checks of the C-ABI library: it loads, exports every symbol include/sv.h declares,
and its host-only entry points (sizes, validation, error strings) behave. No compute calls."""
import ctypes
import os
import re

import pytest

from paper_2604_09562_b200 import sv
import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "sv.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sv_[a-z_0-9]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2604_09562_b200 import build
    if not os.path.exists(sv.LIB_PATH):
        build.build()
    return sv.load()


def test_exports_every_declared_symbol(lib):
    names = _declared()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(sv.EXPORTED)


def test_version_and_strerror(lib):
    assert b"sm_100a" in lib.sv_version()
    for s in range(7):
        assert lib.sv_strerror(s)


def test_query_sizes(lib):
    for name, cfg in synth.CONFIGS.items():
        c = sv.Config.from_any(cfg)
        kv, ws = ctypes.c_size_t(), ctypes.c_size_t()
        assert lib.sv_query_sizes(ctypes.byref(c), ctypes.byref(kv), ctypes.byref(ws)) == sv.SV_OK
        assert kv.value == cfg.n_layers * cfg.n_pages * 2 * cfg.n_kv_heads * cfg.page_size * cfg.head_dim * 2
        assert ws.value % 1024 == 0 and ws.value > 0
    big = sv.Config.from_any(synth.LLAMA)
    kv, ws = ctypes.c_size_t(), ctypes.c_size_t()
    lib.sv_query_sizes(ctypes.byref(big), ctypes.byref(kv), ctypes.byref(ws))
    assert ws.value < 8 << 30          # workspace fits comfortably next to 180 GB of HBM


@pytest.mark.parametrize("field,value", [("n_q_heads", 3), ("head_dim", 96), ("max_depth", 33),
                                         ("max_batch", 0), ("d_model", 100), ("n_kv_heads", 4)])
def test_query_sizes_rejects_bad_config(lib, field, value):
    cfg = synth.LLAMA.with_(**{field: value})
    c = sv.Config.from_any(cfg)
    kv, ws = ctypes.c_size_t(), ctypes.c_size_t()
    assert lib.sv_query_sizes(ctypes.byref(c), ctypes.byref(kv), ctypes.byref(ws)) == sv.SV_EINVAL


def test_host_argument_validation_without_gpu(lib):
    assert lib.sv_create(None, None, None, None, None, None) == sv.SV_EINVAL
    assert lib.sv_verify(None, 1, None, None, None, None, 0, 0, 1.0, None, None, None) == sv.SV_EINVAL
    assert lib.sv_commit(None, None) == sv.SV_EINVAL
    assert lib.sv_stats(None, None, 0) == sv.SV_EINVAL
    assert lib.sv_kv_pack(None, None, 1, 1, 64, 1, 0, None, None) == sv.SV_EINVAL
    c = sv.Config.from_any(synth.TOY)
    assert lib.sv_kv_packed_bytes(ctypes.byref(c), 10) == 1 * 10 * 2 * 2 * 64 * 2 + 16


def test_product_path_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2604_09562_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cpp", ".h", ".cuh")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f


def test_handoff_batch_bytes():
    """sv_kv_slots_bytes: layer x page blocks of every request, then the pending tokens padded to 16 B."""
    import ctypes
    from paper_2604_09562_b200 import sv
    lib = sv.load()
    c = sv.Config.from_any(synth.TOY.with_(n_layers=2))
    blk = 2 * 2 * 64 * 64 * 2
    t = (ctypes.c_int32 * 3)(1, 65, 128)
    assert lib.sv_kv_slots_bytes(ctypes.byref(c), 3, t) == 2 * (1 + 2 + 2) * blk + 16
    assert lib.sv_kv_slots_bytes(ctypes.byref(c), 0, t) == 0


def test_query_sizes_deep_chains(lib):
    """G = 4: chains up to k = 31 (rows-on-lanes attention for (k + 1) G > 64); G = 8 caps at k = 7."""
    kv, ws = ctypes.c_size_t(), ctypes.c_size_t()
    ok = sv.Config.from_any(synth.LLAMA.with_(max_depth=31, max_batch=8, max_slots=8, n_pages=64))
    assert lib.sv_query_sizes(ctypes.byref(ok), ctypes.byref(kv), ctypes.byref(ws)) == sv.SV_OK
    g8 = sv.Config.from_any(synth.LLAMA.with_(n_kv_heads=4, max_depth=7))
    assert lib.sv_query_sizes(ctypes.byref(g8), ctypes.byref(kv), ctypes.byref(ws)) == sv.SV_OK
