"""P=8 vocabulary shards on 4 physical GPUs ("P=8
will run as 8 logical shards on 4 GPUs and be labelled as such").

Each process drives one GPU and two virtual ranks (v = 2r, 2r+1). Every virtual
rank has its own dsdv context and stream and its own exchange buffer. Buffers
on the other GPUs are CUDA-IPC mappings; the two on this GPU are used
directly. A window is one dsdv_shard_verify_peers call per virtual rank, with
P = 8: the stats pass, the three flag rounds, decide + MASS, RESOLVE and the
tokens step. The two virtual ranks of a GPU run on two streams, so their flag
rounds can wait on each other.

Each process reports the device time for its two ranks' windows; rank 0 prints
the max over the GPUs and checks every virtual rank's decisions for equality.
    torchrun --nproc-per-node 4 scripts/p8_on_4gpus.py [steps]"""
import ctypes as C
import json
import os
import sys
from pathlib import Path

import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2511_11733_b200.dsdv import LIB, Verifier, VerifyParams, WindowResult  # noqa: E402
from paper_2511_11733_b200.sharded import (ShardedVerifier, contiguous_slice,  # noqa: E402
                                           slice_bounds)

STEPS = int(sys.argv[1]) if len(sys.argv) > 1 else 10
P = 8
local = int(os.environ.get("LOCAL_RANK", 0))
torch.cuda.set_device(local)
dist.init_process_group("nccl")
rank, world = dist.get_rank(), dist.get_world_size()
assert world * 2 == P, "run with 4 processes"
B, G, V = 256 * P, 8, 128256
dev = torch.device("cuda", local)
vs = [Verifier(local), Verifier(local)]
svs = [ShardedVerifier(v) for v in vs]
draft_f, target_f = vs[0].synth_logits(B, G, V, torch.bfloat16, logits_seed=42)
p = VerifyParams(gamma=G, tau=0.2, seed=1)
tokens = vs[0].draft_sample(draft_f, p, vocab=V)
mine = [2 * rank, 2 * rank + 1]
slices = []
for v in mine:
    lo, n = slice_bounds(V, P, v)
    slices.append((lo, n, contiguous_slice(draft_f, lo, n), contiguous_slice(target_f, lo, n)))
del draft_f, target_f
torch.cuda.synchronize()

# exchange buffers: one per virtual rank, IPC handles swapped once
_, size = ShardedVerifier.exchange_layout(B, G, p.top_m)
stride = -(-size // 256) * 256
nbytes = 2 * P * stride + 8 * P
own, handles = [], []
for v in vs:
    ptr = C.c_void_p()
    v._check(LIB.dsdv_dev_alloc(v._h, nbytes, C.byref(ptr)))
    h = (C.c_uint8 * 64)()
    v._check(LIB.dsdv_ipc_handle(v._h, ptr, h))
    own.append(ptr.value)
    handles.append(list(bytearray(h)))
mine_h = torch.tensor(handles, dtype=torch.uint8, device=dev)
all_h = torch.empty((world, 2, 64), dtype=torch.uint8, device=dev)
dist.all_gather_into_tensor(all_h, mine_h)
all_h = all_h.cpu()
bases, opened = [], []
for q in range(P):
    r, k = divmod(q, 2)
    if r == rank:
        bases.append(own[k])
        continue
    h = (C.c_uint8 * 64)(*all_h[r, k].tolist())
    ptr = C.c_void_p()
    vs[0]._check(LIB.dsdv_ipc_open(vs[0]._h, h, C.byref(ptr)))
    opened.append(ptr.value)
    bases.append(ptr.value)
dist.barrier()

streams = [torch.cuda.Stream(dev), torch.cuda.Stream(dev)]
outs = [WindowResult.allocate(B, G, dev, True, records=True) for _ in mine]
cbases = (C.c_void_p * P)(*bases)


def window(epoch):
    for k in range(2):
        lo, n, d, t = slices[k]
        p.window = epoch
        cp = svs[k]._cp(p, d, t, tokens, V, lo, n)
        vs[k]._check(LIB.dsdv_shard_verify_peers(
            vs[k]._h, C.byref(cp), d.data_ptr(), t.data_ptr(), tokens.data_ptr(), P, mine[k],
            cbases, stride, epoch, int(10e9), C.byref(outs[k]._c), streams[k].cuda_stream))


epoch = 1
for _ in range(3):
    window(epoch)
    epoch += 1
torch.cuda.synchronize()
dist.barrier()
ev = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(2)]
for k in range(2):
    ev[k][0].record(streams[k])
for _ in range(STEPS):
    window(epoch)
    epoch += 1
for k in range(2):
    ev[k][1].record(streams[k])
torch.cuda.synchronize()
ms = max(ev[k][0].elapsed_time(ev[k][1]) for k in range(2)) / STEPS
t = torch.tensor([ms], device=dev)
dist.all_reduce(t, op=dist.ReduceOp.MAX)
ms = float(t.item())
# every virtual rank holds the same decisions
ks = torch.stack([o.accepted_count for o in outs] + [o.extra_token for o in outs])
gathered = torch.empty((world, *ks.shape), dtype=ks.dtype, device=dev)
dist.all_gather_into_tensor(gathered, ks.contiguous())
same = bool((gathered[:, :2] == gathered[0, 0]).all() and (gathered[:, 2:] == gathered[0, 2]).all())
bad = int(sum(int((o.status != 0).sum()) for o in outs))
parity = None
if rank == 0:
    # the last window against the fp64 oracle over the unsharded rows
    from oracle.oracle_lib import Oracle, window_uniforms
    from tests.parity_util import compare_batch, host_logits
    crit = Oracle.crit(p.ratio_limit, p.gap_limit, p.overlap_floor, p.top_m)
    gpu = outs[0].to_host()
    d_full, t_full = vs[0].synth_logits(B, G, V, torch.bfloat16, logits_seed=42)
    dh, th = host_logits(d_full), host_logits(t_full)
    del d_full, t_full
    ref = Oracle().verify_batch(dh, th, tokens.cpu().numpy(), [(p.tau, crit)],
                                window_uniforms(1, epoch - 1, B, G), V, all_positions=True)[0]
    rep = compare_batch(ref, gpu)
    parity = {"window": epoch - 1, "sequences": rep.sequences, "mismatches": len(rep.mismatches),
              "eps_events": rep.eps_events}
if rank == 0:
    print(json.dumps({
        "config": "C4 at P=8: 8 logical shards on 4 GPUs (2 per GPU, one stream each), "
                  "V=128256 (16032 ids per shard), B=2048, gamma=8, bf16",
        "ms_per_window": ms, "verified_tokens_per_s": B * G / (ms * 1e-3), "gpus": world,
        "logical_shards": P, "steps": STEPS, "all_ranks_equal": same, "status_errors": bad,
        "mean_accepted_k": float(outs[0].accepted_count.float().mean()), "parity": parity,
        "note": "per GPU: two P=8 ranks' work (the stats passes of both share the GPU)"}),
        flush=True)
torch.cuda.synchronize()
for ptr in opened:
    LIB.dsdv_ipc_close(vs[0]._h, C.c_void_p(ptr))
dist.barrier()
for k, v in enumerate(vs):
    LIB.dsdv_dev_free(v._h, C.c_void_p(own[k]))
dist.destroy_process_group()
