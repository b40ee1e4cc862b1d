"""The N=8 bench shape (B=2048, 8 vocabulary slices) in one process: the
collective-free peer protocol equals the gathered path bit for bit (development
aid; run on one GPU)."""
import torch, sys
sys.path.insert(0, '/root/repo')
from paper_2511_11733_b200.dsdv import Verifier, VerifyParams
from paper_2511_11733_b200.sharded import shard_slices, shard_slices_peer
v = Verifier(0)
B, G, V = 2048, 8, 128256
d, t = v.synth_logits(B, G, V, torch.bfloat16, logits_seed=42)
p = VerifyParams(gamma=G, tau=0.2, seed=1)
tok = v.draft_sample(d, p, vocab=V)
a = shard_slices(v, d, t, tok, p, V, 8).to_host()
b = shard_slices_peer(v, d, t, tok, p, V, 8, epoch=5).to_host()
bad = [k for k in a if not (torch.equal(a[k], b[k]) or (a[k].is_floating_point() and torch.equal(a[k].nan_to_num(7.0), b[k].nan_to_num(7.0))))]
print("P=8 B=2048 peer vs gathered:", "OK" if not bad else bad, "mean k", a["accepted_count"].float().mean().item(), "status errors", int((a["status"] != 0).sum()))
