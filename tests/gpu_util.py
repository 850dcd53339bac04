"""Helpers for the -m gpu parity tests: build a lane from synth inputs, read taps,
compare bf16 tensors in ulps. Expected values always come from `oracle/`."""
import numpy as np
import torch

import synth
from paper_2604_09562_b200 import sv


def bf16_ulp_diff(a, b):
    """|a - b| in bf16 ulps (ordered-integer distance), a and b torch bf16 tensors."""
    def ordered(t):
        i = t.contiguous().view(torch.int16).to(torch.int32)
        return torch.where(i < 0, -32768 - i, i)
    return (ordered(a) - ordered(b)).abs()


def to_bf16(x):
    """fp64 numpy array of bf16 values -> torch bf16 (exact)."""
    return torch.from_numpy(np.ascontiguousarray(x)).to(torch.bfloat16)


def f64(t):
    return t.detach().cpu().to(torch.float64).numpy()


class Setup:
    """A lane + matching oracle inputs: requests with synthetic context KV."""

    def __init__(self, cfg, ctx_lens, seed=0, norm_one=False, weights=None, embed_std=1.0, std=0.02):
        self.cfg = cfg
        self.w = weights if weights is not None else synth.model_weights(cfg, seed=seed, norm_one=norm_one,
                                                                          embed_std=embed_std, std=std)
        self.wd = {k: v.cuda() for k, v in self.w.items()}
        self.lane = sv.Lane(cfg, self.wd)
        self.lane.set_taps(True)                    # the stage tests read every intermediate
        self.ctx = []
        for i, n in enumerate(ctx_lens):
            k, v = synth.context_kv(cfg, n, seed=1000 + 17 * seed + i)
            pend = int(synth.random_tokens(1, cfg.vocab, seed=2000 + i)[0])
            rid = (i + 1) * 0x1_0000_0001 + seed
            self.lane.append_kv(i, rid, k.cuda(), v.cuda(), pend)
            self.ctx.append(dict(k=k, v=v, pending=pend, rid=rid, L=n))
        self._wnp = None

    @property
    def wnp(self):
        if self._wnp is None:
            self._wnp = {k: (v.to(torch.float32).numpy()) for k, v in self.w.items()}
        return self._wnp

    def tap(self, name, dtype, shape):
        torch.cuda.synchronize()
        return self.lane.tap(name, dtype, shape).cpu().clone()
