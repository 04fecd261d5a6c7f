"""The N>1 host path with real ranks (world_size 2, gloo, CPU): per-rank layouts, the packed
index all-gather (TorchDistExchange) and its reassembly into the global (sender-major)
content order, remote-key resolution, ledger.  The CUDA kernels are covered by the GPU
tests; here the pack/unpack arithmetic is the oracle's (CPU)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import astra_oracle as O


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _unpack(words: np.ndarray, count: int, bits: int) -> np.ndarray:
    v = words.astype(np.uint64)
    out = np.empty(count, dtype=np.int64)
    for i in range(count):
        b = i * bits
        w, off = divmod(b, 32)
        pair = int(v[w]) | ((int(v[w + 1]) << 32) if w + 1 < len(v) else 0)
        out[i] = (pair >> off) & ((1 << bits) - 1)
    return out


def _worker(rank, world, port, T, B, K, result_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2505_19342_b200.cluster import CommsLedger, partition_tokens
        from paper_2505_19342_b200.layout import resolve_keys, sp_layout
        from paper_2505_19342_b200.runtime import TorchDistExchange
        from paper_2505_19342_b200.vq import index_bits
        plan = partition_tokens(T, world)
        owners = list(range(world))
        bits = index_bits(K)
        comm = TorchDistExchange()
        mine = sp_layout(T, plan.ranges, B, [rank], owners)
        virt = sp_layout(T, plan.ranges, B, list(range(world)), owners)
        codes = np.random.default_rng(7).integers(0, K, size=int(virt.gofs[-1]))
        # this rank encodes its shard: tokens (b, r) in order == its slice of the global order
        lo, hi = int(mine.gofs[rank]), int(mine.gofs[rank + 1])
        own = codes[lo:hi]
        wmax = (B * max(plan.shard_sizes()) * bits + 31) // 32
        words = np.zeros(wmax, np.uint32)
        packed = O.pack_indices(own, bits)
        words[:len(packed)] = packed
        send = torch.from_numpy(words.view(np.int32).copy())
        recv = torch.zeros(world * wmax, dtype=torch.int32)
        comm.all_gather(recv, send)
        allw = recv.numpy().view(np.uint32)
        got = np.concatenate([_unpack(allw[e * wmax:(e + 1) * wmax],
                                      B * plan.shard_sizes()[e], bits) for e in range(world)])
        ok_codes = bool(np.array_equal(got, codes))
        # remote keys resolve to the same codes as the single-GPU (virtual) layout's
        rk = resolve_keys(mine.key_map, got)
        vk = resolve_keys(virt.key_map, codes)
        ok_keys = True
        for b in range(B):
            s_m = mine.segs[b]
            s_v = virt.segs[rank * B + b]
            km = rk[s_m[4]:s_m[4] + s_m[5]]
            kv = vk[s_v[4]:s_v[4] + s_v[5]]
            # local keys: same token position; remote keys: same code
            for a, c in zip(km, kv):
                if (a < 0) != (c < 0):
                    ok_keys = False
                elif a < 0:
                    ok_keys &= bool(a == c)
                else:
                    ok_keys &= bool(mine.row_pos[a] == virt.row_pos[c])
        led = CommsLedger()
        led.record_exchange(0, [B * s * bits for s in plan.shard_sizes()])
        result_q.put((rank, ok_codes, ok_keys, led.total_bits_sent(), mine.rows))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("T,B,K", [(11, 3, 1024), (196, 2, 1024), (9, 1, 5)])
def test_two_rank_exchange_and_layout(T, B, K):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, T, B, K, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    for rank, ok_codes, ok_keys, bits_sent, rows in res:
        assert ok_codes and ok_keys, (rank, ok_codes, ok_keys)
    assert res[0][3] == res[1][3]
    sizes = [e - s for s, e in O.partition_tokens(T, 2)]
    assert res[0][4] == B * (sizes[0] + 1) and res[1][4] == B * (sizes[1] + 1)
