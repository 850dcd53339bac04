"""a9 hand-off rates on one B200 at the c4 shape (BASELINE configs[3]: 32 requests x 8192-token
prompts, Llama-3-8B KV, 1 layer = 32 MiB per request, 1.07 GB per batch fill):

  pack     sv_kv_pack_slot   committed pages of a prefill lane -> wire format     (read + write)
  append   sv_kv_append_packed  wire format -> freshly popped pages of a decode lane (read + write)
  loopback sv_kv_loopback_append  NCCL send-to-self + receive into staging + scatter (one GPU:
           measures NCCL's on-device path, not NVLink; the 2-GPU transfer needs two GPUs)

CUDA-event times per batch fill; GB/s counts the wire bytes once (the data moved per fill)."""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch

import synth
from paper_2604_09562_b200 import sv

B, N = 32, 8192
cfg = synth.LLAMA.with_(n_pages=B * (N // 64 + 2), max_slots=B, max_batch=B, max_pos=N + 128, ffn_dim=0)
w = {k: v.cuda() for k, v in synth.model_weights(cfg, seed=0).items()}
pre, dec = sv.Lane(cfg, w), sv.Lane(cfg, w)
nb = pre.packed_bytes(N)
for i in range(B):
    k, v = synth.context_kv(cfg, N, seed=10 + i, device="cuda")
    pre.append_kv(i, 100 + i, k, v, 7)
packed = [torch.empty(nb, dtype=torch.uint8, device="cuda") for _ in range(B)]
staging = torch.empty(nb, dtype=torch.uint8, device="cuda")
comm = sv.nccl_comm_init(1, sv.nccl_unique_id(), 0)


def timed(fn, reps=3):
    best = None
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1)
        best = t if best is None else min(best, t)
    return best


def pack():
    for i in range(B):
        pre.kv_pack_slot(i, N, packed[i])


def append():
    for i in range(B):
        dec.release(i)
    for i in range(B):
        dec.kv_append_packed(i, 100 + i, N, packed[i])


def loopback():
    for i in range(B):
        dec.release(i)
    for i in range(B):
        dec.kv_loopback_append(i, 100 + i, N, packed[i], staging, 0, comm)


total = B * nb
for name, fn in (("pack", pack), ("append", append), ("loopback", loopback)):
    ms = timed(fn)
    print(f"{name:8s}: {B} x {nb / 2**20:.1f} MiB = {total / 1e9:.2f} GB in {ms:.2f} ms = {total / ms / 1e6:.0f} GB/s "
          f"({2 * total / ms / 1e6:.0f} GB/s read + write)", flush=True)
sv.nccl_comm_destroy(comm)
