"""Measured-communication model (paper_2505_19342_b200.comms).

* with an analytic link it reproduces the reference's frozen numbers (the pinned values of
  /root/reference/pkg/tests/test_comms.py:81-87 and :169-177, comms.py:118-209);
* the exact wire payload equals the runtime's packed all-gather buffer (word-padded, largest
  shard) and is never below the ledger's bit count;
* measure_allgather + fit_link run over a real world-size-2 gloo group (the NCCL path is the
  same call on CUDA tensors)."""

import os
import socket
from fractions import Fraction

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2505_19342_b200 import comms as C


def _cfg(**kw):
    base = dict(layers=12, hidden=768, tokens=1024, devices=4,
                bandwidth_bps=Fraction(10) * 10**6, codebook_size=1024, groups=1,
                precision_bits=32)
    base.update(kw)
    return C.CommsConfig(**base)


def test_frozen_reference_row():
    rows = C.speedup_table_measured(_cfg(seconds_per_flop=5e-13), [C.MethodSpec("astra")],
                                    devices=[4], tokens=[1024], exact_wire=False)
    lines = C.bench_csv(rows).splitlines()
    assert lines[0] == ",".join(C.BENCH_COLUMNS)
    assert lines[1] == "astra,1,10,4,1024,0.028991,0.009216,0.038207,2.78222"


def test_sp_and_tp_comm_times_match_reference_formulas():
    assert C.comm_time(_cfg(), C.MethodSpec("sp")) == pytest.approx(22.6492416, rel=1e-12)
    # tp: two ring all-reduces per layer, 2 (N-1)/N V / B each (comms.py:139-144)
    v_bits = 1024 * 768 * 32
    want = 2 * 12 * (2 * 3 / 4 * v_bits / 10e6)
    assert C.comm_time(_cfg(), C.MethodSpec("tp")) == pytest.approx(want, rel=1e-12)
    assert C.comm_time(_cfg(devices=1), C.MethodSpec("astra")) == 0.0


def test_link_model_latency_term():
    link = C.LinkModel(alpha_s=2e-6, beta_Bps=100e9, source="test")
    # (N-1) * (alpha + S / beta) per collective, one per layer
    got = C.comm_time(_cfg(devices=8), C.MethodSpec("astra"), link, batch=64, exact_wire=True)
    s = C.astra_wire_bytes(1024, 8, 1, 1024, batch=64)
    assert got == pytest.approx(12 * 7 * (2e-6 + s / 100e9))


@pytest.mark.parametrize("T,N,G,K,B", [(196, 4, 1, 1024, 64), (196, 3, 1, 1024, 1),
                                       (576, 8, 16, 1024, 32), (1024, 4, 1, 1024, 8),
                                       (7, 2, 4, 5, 3)])
def test_wire_bytes_match_runtime_buffer_and_ledger(T, N, G, K, B):
    from paper_2505_19342_b200.cluster import partition_tokens
    from paper_2505_19342_b200.vq import index_bits
    plan = partition_tokens(T, N)
    bits = index_bits(K)
    wmax = (B * max(plan.shard_sizes()) * G * bits + 31) // 32      # runtime send buffer
    assert C.astra_wire_bytes(T, N, G, K, B) == 4 * wmax
    ledger_bits = B * max(plan.shard_sizes()) * G * bits
    assert 8 * C.astra_wire_bytes(T, N, G, K, B) - ledger_bits in range(0, 32)


def test_measured_compute_overrides_flop_profile():
    comp = {("single", 1, 196): 4.0e-3, ("astra", 4, 196): 1.9e-3}
    link = C.LinkModel(1e-6, 200e9, "test")
    rows = C.speedup_table_measured(_cfg(tokens=196), [C.MethodSpec("astra"), C.MethodSpec("sp")],
                                    devices=[4], tokens=[196], link=link, compute_s=comp,
                                    batch=64)
    a, sp = rows
    assert a["compute_s"] == 1.9e-3 and a["speedup"] == pytest.approx(4.0e-3 / a["total_s"])
    assert sp["compute_s"] == C.compute_time(_cfg(tokens=196), C.MethodSpec("sp"))
    assert a["bandwidth_mbps"] == pytest.approx(200e9 * 8 / 1e6)


def test_fit_link_recovers_alpha_beta():
    alpha, beta = 3e-6, 50e9
    samples = [(n, s, (n - 1) * (alpha + s / beta)) for n in (2, 4, 8) for s in (1e3, 1e5, 1e7)]
    link = C.fit_link(samples)
    assert link.alpha_s == pytest.approx(alpha, rel=1e-6)
    assert link.beta_Bps == pytest.approx(beta, rel=1e-6)
    with pytest.raises(ValueError):
        C.fit_link([(1, 100, 0.0)])


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        samples = C.measure_allgather([3920, 1 << 16, 1 << 20], reps=5, warmup=1)
        if rank == 0:
            q.put(samples)
    finally:
        dist.destroy_process_group()


def test_measure_allgather_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    samples = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [s[0] for s in samples] == [2, 2, 2]
    assert [s[1] for s in samples] == [3920, 1 << 16, 1 << 20]
    assert all(s[2] > 0 for s in samples)
    link = C.fit_link(samples, "gloo")
    assert link.alpha_s >= 0 and link.beta_Bps > 0
