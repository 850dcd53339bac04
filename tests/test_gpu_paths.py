"""The library's alternative kernel paths (kept as in-library cross-checks, selected per lane at
sv_create by environment): SIMT / rows-on-lanes attention and the SIMT / token-major 1-SM / 2-SM
GEMMs, through the same teacher-forced stage parity as the default path (tests/test_gpu_parity.py)
at Llama shape on a small request set."""
import os

import pytest

import synth

from gpu_util import Setup
from test_gpu_parity import run_and_check

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("env", [{"SV_ATTN": "simt"}, {"SV_ATTN": "tc1"}, {"SV_GEMM": "simt"}, {"SV_GEMM": "tc1"},
                                 {"SV_GEMM": "tc2"}])
def test_alternative_paths_stage_parity(env):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        cfg = synth.LLAMA.with_(n_pages=96, max_slots=4, max_batch=4, max_pos=2048)
        S = Setup(cfg, [300, 1100, 64, 700], seed=23)
        slots, depths = [0, 1, 2, 3], [8, 3, 0, 5]
        drafts = synth.random_tokens(sum(depths), cfg.vocab, seed=24)
        rep, _, _ = run_and_check(S, slots, depths, drafts, "greedy")
        print(env, rep)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
