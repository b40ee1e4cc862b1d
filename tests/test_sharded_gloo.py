"""Host-side logic of the vocabulary-sharded verifier on CPU (no GPU): two
gloo ranks exchange per-slice partial statistics through sharded.TorchComm in
the layout dsdv_shard_stats produces, and the shard-order merge
(csrc/shard.cu: log-sum-exp of the slice normalisers, P-way (value desc,
id asc) merge of the slice top-m lists, ascending-id ownership of the inverse
CDF) reproduces the unsharded fp64 oracle on the whole row."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2511_11733_b200.sharded import TorchComm, slice_bounds


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _slice_stats(lt, ld, lo, n, y, M):
    """Partial record + top lists of one slice (the quantities of write_partial)."""
    t, d = lt[lo:lo + n], ld[lo:lo + n]
    mt, md = t.max(), d.max()
    rec = np.array([mt, np.log(np.exp(t - mt).sum()), md, np.log(np.exp(d - md).sum()),
                    lt[y] if lo <= y < lo + n else np.nan, float(lo <= y < lo + n)])
    def top(v):
        order = sorted(range(n), key=lambda i: (-v[i], i))[:M]
        ids = np.full(M, -1, np.int64)
        vals = np.full(M, -np.inf)
        ids[:len(order)] = [lo + i for i in order]
        vals[:len(order)] = [v[i] for i in order]
        return vals, ids
    return rec, top(t), top(d)


def _merge_top(vals, ids, M):
    cand = [(-v, i) for vv, ii in zip(vals, ids) for v, i in zip(vv, ii) if i >= 0]
    return [i for _, i in sorted(cand)[:M]]


def _worker(rank, world, port, V, M, result):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = TorchComm()
        rng = np.random.default_rng(7)
        lt = rng.normal(size=V) * 3
        ld = 0.7 * lt + rng.normal(size=V)
        y = int(rng.integers(0, V))
        lo, n = slice_bounds(V, world, rank)
        rec, (tv, ti), (dv, di) = _slice_stats(lt, ld, lo, n, y, M)
        recs = comm.all_gather(torch.from_numpy(rec)).numpy()
        tvs = comm.all_gather(torch.from_numpy(tv)).numpy()
        tis = comm.all_gather(torch.from_numpy(ti)).numpy()
        dvs = comm.all_gather(torch.from_numpy(dv)).numpy()
        dis = comm.all_gather(torch.from_numpy(di)).numpy()
        # merged normalisers vs the whole row
        lse_t = np.logaddexp.reduce(recs[:, 0] + recs[:, 1])
        lse_d = np.logaddexp.reduce(recs[:, 2] + recs[:, 3])
        full_t = lt.max() + np.log(np.exp(lt - lt.max()).sum())
        full_d = ld.max() + np.log(np.exp(ld - ld.max()).sum())
        owners = recs[:, 5].sum()
        lt_y = recs[recs[:, 5] == 1][0, 4]
        top_t = _merge_top(tvs, tis, M)
        top_d = _merge_top(dvs, dis, M)
        ref_t = sorted(range(V), key=lambda i: (-lt[i], i))[:M]
        ref_d = sorted(range(V), key=lambda i: (-ld[i], i))[:M]
        # inverse CDF over ascending ids: the owner of T by cumulative slice mass
        p = np.exp(lt - full_t)
        masses = comm.all_gather(torch.tensor([p[lo:lo + n].sum()])).numpy()[:, 0]
        u = 0.6180339887
        T = u * masses.sum()
        owner = int(np.searchsorted(np.cumsum(masses), T, side="right"))
        tok = torch.tensor([-1])
        if owner == rank:
            local = np.cumsum(p[lo:lo + n]) + (np.cumsum(masses)[rank] - masses[rank])
            tok[0] = lo + int(np.searchsorted(local, T, side="right"))
        comm.all_reduce_max(tok)
        ref_tok = int(np.searchsorted(np.cumsum(p), u * p.sum(), side="right"))
        result[rank] = (abs(lse_t - full_t) < 1e-12 and abs(lse_d - full_d) < 1e-12
                        and owners == 1 and lt_y == lt[y] and top_t == ref_t and top_d == ref_d
                        and int(tok[0]) == ref_tok)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_exchange_reproduces_the_whole_row(world):
    mp_ctx = mp.get_context("spawn")
    result = mp_ctx.Manager().dict()
    port = _free_port()
    procs = [mp_ctx.Process(target=_worker, args=(r, world, port, 4099, 10, result))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert all(result[r] for r in range(world)), dict(result)


def test_slice_bounds_cover_the_vocabulary():
    for V in (128256, 151936, 32000, 1000):
        for P in (2, 3, 4, 8):
            parts = [slice_bounds(V, P, r) for r in range(P)]
            assert parts[0][0] == 0
            assert sum(n for _, n in parts) == V
            for (lo, n), (lo2, _) in zip(parts, parts[1:]):
                assert lo + n == lo2 and lo2 % 8 == 0


def test_peer_exchange_layout():
    """Slot layout of the collective-free window: records, top lists, masses and
    tokens aligned for their element types and inside one stride; the flag array
    sits after both alternating sets (host arithmetic only, no device)."""
    from paper_2511_11733_b200.sharded import PeerExchange, ShardedVerifier
    for B, G, M in ((256, 8, 10), (1024, 16, 6), (3, 1, 1)):
        (o_rec, o_tv, o_ti, o_mass, o_tok), size = ShardedVerifier.exchange_layout(B, G, M)
        (p_rec, p_tv, p_ti), psize = ShardedVerifier.packed_layout(B, G, M)
        assert (o_rec, o_tv, o_ti) == (p_rec, p_tv, p_ti)
        assert o_mass >= psize and o_mass % 8 == 0 and o_tok == o_mass + 8 * B
        assert size == o_tok + 4 * B
        for P in (2, 4, 8):
            bases = [(q + 1) << 32 for q in range(P)]
            ex = PeerExchange(None, P, P - 1, size, bases=bases)
            assert ex.stride >= size and ex.stride % 256 == 0
            for w in (1, 2):
                sets = ex.set_bases(w)
                assert [s - b for s, b in zip(sets, bases)] == [(w & 1) * P * ex.stride] * P
            # dsdv_peer_signal / _wait address flag q at flag_base + P * stride + 8 q
            assert [f + P * ex.stride - b for f, b in zip(ex.flag_bases(), bases)] == \
                [2 * P * ex.stride] * P
            assert ex.bytes == 2 * P * ex.stride + 8 * P
