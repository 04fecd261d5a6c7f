"""Communication model of the Astra exchange, measured instead of assumed.

The reference prices communication analytically (`seqvq.comms`, comms.py:1-262): an
all-gather of per-device shards of S bits over a ring costs ``rounds * ((N-1) S / B +
(N-1) * msg_latency)`` (comms.py:118-124), Astra sends ``layers * G * ceil(log2 K)`` bits per
token (comms.py:91-109), and compute is a FLOP count times a seconds-per-FLOP profile
(comms.py:152-189).  This module keeps that model and its CSV schema (``BENCH_COLUMNS``,
comms.py:23-24, 212-262) but lets both inputs come from measurements on the box:

* :func:`measure_allgather` times the real packed-index exchange of the runtime
  (``all_gather_into_tensor`` over torch.distributed — NCCL over NVLink/NVSwitch on a GPU
  box, gloo on CPU), device-timed and max-over-ranks like the bench;
* :func:`fit_link` fits the ring model's per-hop latency ``alpha`` and bandwidth ``beta`` to
  those samples (least squares on ``t = (N-1) * (alpha + S / beta)``);
* :func:`astra_wire_bytes` is the exact payload the runtime puts on the wire per rank and
  layer — the LSB-first packed codes in 32-bit words, padded to the largest shard
  (cluster.py:79-128 / runtime exchange), not the model's fractional bits;
* :func:`speedup_table_measured` produces the reference's sweep rows with ``comm_s`` from the
  fitted link and, when given, ``compute_s`` from measured per-rank forward times.

With ``LinkModel.from_analytic(bandwidth_bps, msg_latency_s)`` the functions reproduce the
reference's analytic numbers (tests pin its frozen rows), so the two can be compared column
by column.
"""

from __future__ import annotations

import csv
import io
import math
import time
from dataclasses import dataclass, replace
from fractions import Fraction

from .vq import index_bits

METHODS = ("single", "astra", "sp", "tp", "bp_ag", "bp_sp")
BENCH_COLUMNS = ("method", "Nb", "bandwidth_mbps", "devices", "tokens",
                 "compute_s", "comm_s", "total_s", "speedup")
DEFAULT_SECONDS_PER_FLOP = 5e-13      # the reference's laptop-class anchor (comms.py:26-28)


@dataclass(frozen=True)
class CommsConfig:
    """Same fields and validation as the reference's CommsConfig (comms.py:31-62)."""
    layers: int
    hidden: int
    tokens: int
    devices: int
    bandwidth_bps: Fraction | int
    codebook_size: int = 1024
    groups: int = 1
    precision_bits: int = 32
    msg_latency_s: Fraction | float = 0
    heads: int = 12
    mlp_expansion: int = 4
    seconds_per_flop: float = DEFAULT_SECONDS_PER_FLOP
    bp_ag_volume_coeff: Fraction | int = 1
    bp_sp_volume_coeff: Fraction | int = 2
    bp_ag_compute_coeff: float = 1.2
    bp_sp_compute_coeff: float = 1.0

    def __post_init__(self):
        if min(self.layers, self.hidden, self.tokens, self.devices) < 1:
            raise ValueError("layers/hidden/tokens/devices must be positive")
        if Fraction(self.bandwidth_bps) <= 0:
            raise ValueError("bandwidth must be positive")
        if self.precision_bits < 1:
            raise ValueError("precision must be at least one bit")
        if Fraction(self.msg_latency_s) < 0:
            raise ValueError("per-message latency cannot be negative")


@dataclass(frozen=True)
class MethodSpec:
    method: str
    nb: int = 1

    def __post_init__(self):
        if self.method not in METHODS:
            raise ValueError(f"unknown method {self.method!r}")
        if self.nb < 1:
            raise ValueError("Nb must be at least 1")


@dataclass(frozen=True)
class LinkModel:
    """Ring all-gather cost ``(N-1) * (alpha_s + shard_bytes / beta_Bps)`` per collective.

    ``source`` says where the numbers came from ("analytic", "nccl", "gloo", ...)."""
    alpha_s: float
    beta_Bps: float
    source: str = "analytic"

    @staticmethod
    def from_analytic(bandwidth_bps, msg_latency_s=0.0) -> "LinkModel":
        return LinkModel(float(msg_latency_s), float(Fraction(bandwidth_bps)) / 8.0, "analytic")

    @property
    def bandwidth_mbps(self) -> float:
        return self.beta_Bps * 8.0 / 1e6

    def allgather_s(self, devices: int, shard_bytes: float, rounds: int = 1) -> float:
        if devices == 1:
            return 0.0
        return rounds * (devices - 1) * (self.alpha_s + shard_bytes / self.beta_Bps)


def astra_wire_bytes(tokens: int, devices: int, groups: int, codebook_size: int,
                     batch: int = 1) -> int:
    """Bytes one rank contributes to one layer's exchange: B * T_max * G codes of
    ceil(log2 K) bits, LSB-first in 32-bit words, T_max = the largest shard (the payload is
    padded to it so the all-gather is uniform; true lengths are static)."""
    t_max = -(-tokens // devices)
    bits = batch * t_max * groups * index_bits(codebook_size)
    return 4 * (-(-bits // 32))


def _shard_bytes(cfg: CommsConfig, spec: MethodSpec, batch: int, exact_wire: bool) -> tuple:
    """(shard bytes per rank per collective, collectives) for the all-gather methods."""
    n = cfg.devices
    full_row_bytes = Fraction(cfg.hidden * cfg.precision_bits, 8)
    shard_tokens = Fraction(cfg.tokens, n)
    if spec.method == "astra":
        if exact_wire:
            return Fraction(astra_wire_bytes(cfg.tokens, n, cfg.groups, cfg.codebook_size,
                                             batch)), cfg.layers
        return batch * shard_tokens * cfg.groups * Fraction(index_bits(cfg.codebook_size), 8), \
            cfg.layers
    if spec.method == "sp":
        return batch * shard_tokens * full_row_bytes, cfg.layers
    if spec.method == "bp_ag":
        return batch * shard_tokens * full_row_bytes * Fraction(cfg.bp_ag_volume_coeff), spec.nb
    if spec.method == "bp_sp":
        return batch * shard_tokens * full_row_bytes * Fraction(cfg.bp_sp_volume_coeff), spec.nb
    raise ValueError(spec.method)


def comm_time(cfg: CommsConfig, spec: MethodSpec, link: LinkModel | None = None,
              batch: int = 1, exact_wire: bool = False) -> float:
    """Per-forward communication seconds (comms.py:127-151 structure) on ``link`` (default:
    the config's own bandwidth / latency, i.e. the reference's analytic number).
    ``exact_wire`` prices Astra's real word-padded payload instead of fractional bits."""
    link = link or LinkModel.from_analytic(cfg.bandwidth_bps, cfg.msg_latency_s)
    n = cfg.devices
    if spec.method == "single" or n == 1:
        return 0.0
    if spec.method == "tp":   # two ring all-reduces of the full activation per layer
        vol = Fraction(batch * cfg.tokens * cfg.hidden * cfg.precision_bits, 8)
        per = 2 * float(Fraction(n - 1, n) * vol) / link.beta_Bps + 2 * (n - 1) * link.alpha_s
        return 2 * cfg.layers * per
    shard, rounds = _shard_bytes(cfg, spec, batch, exact_wire)
    return link.allgather_s(n, float(shard), rounds)


def _layer_flops(cfg: CommsConfig, tokens_per_device: Fraction) -> Fraction:
    d, t = cfg.hidden, tokens_per_device
    return 8 * t * d * d + 4 * t * cfg.tokens * d + 4 * t * d * (cfg.mlp_expansion * d)


def compute_time(cfg: CommsConfig, spec: MethodSpec) -> float:
    """Analytic per-forward compute seconds (comms.py:164-189)."""
    n = cfg.devices
    base = cfg.layers * _layer_flops(cfg, Fraction(cfg.tokens))
    shard = cfg.layers * _layer_flops(cfg, Fraction(cfg.tokens, n))
    flops = {
        "single": lambda: base,
        "tp": lambda: base / n,
        "sp": lambda: shard,
        "astra": lambda: shard + cfg.layers * 2 * Fraction(cfg.tokens, n) * cfg.codebook_size
        * cfg.hidden,
        "bp_ag": lambda: base / n * Fraction(cfg.bp_ag_compute_coeff).limit_denominator(10**6),
        "bp_sp": lambda: base / n * Fraction(cfg.bp_sp_compute_coeff).limit_denominator(10**6),
    }[spec.method]()
    return float(flops) * cfg.seconds_per_flop


def speedup_table_measured(cfg: CommsConfig, specs: list, devices: list, tokens: list,
                           link: LinkModel | None = None, compute_s: dict | None = None,
                           batch: int = 1, exact_wire: bool = True) -> list:
    """The reference's sweep (comms.py:193-209) with measured inputs: ``comm_s`` on ``link``
    (``bandwidth_mbps`` reports its fitted bandwidth) and, for (method, devices, tokens) keys
    present in ``compute_s``, the measured per-rank forward seconds instead of the FLOP
    profile.  ``speedup`` is against ``compute_s[("single", 1, tokens)]`` when measured."""
    rows = []
    for t in tokens:
        for n in devices:
            c = replace(cfg, tokens=t, devices=n)
            lk = link or LinkModel.from_analytic(c.bandwidth_bps, c.msg_latency_s)

            def comp(spec, c=c, n=n, t=t):
                if compute_s is not None and (spec.method, n, t) in compute_s:
                    return float(compute_s[(spec.method, n, t)])
                return compute_time(c, spec)

            if compute_s is not None and ("single", 1, t) in compute_s:
                single = float(compute_s[("single", 1, t)])
            else:
                single = compute_time(c, MethodSpec("single"))
            for spec in specs:
                cs = comp(spec)
                ms = comm_time(c, spec, lk, batch, exact_wire and spec.method == "astra")
                rows.append({"method": spec.method, "Nb": spec.nb,
                             "bandwidth_mbps": lk.bandwidth_mbps, "devices": n, "tokens": t,
                             "compute_s": cs, "comm_s": ms, "total_s": cs + ms,
                             "speedup": single / (cs + ms)})
    return rows


def _fmt(v) -> str:
    return format(v, ".6g") if isinstance(v, float) else str(v)


def bench_csv(rows: list) -> str:
    """Same CSV as the reference's bench_csv (comms.py:218-225)."""
    buf = io.StringIO()
    w = csv.writer(buf, lineterminator="\n")
    w.writerow(BENCH_COLUMNS)
    for r in rows:
        w.writerow([_fmt(r[c]) for c in BENCH_COLUMNS])
    return buf.getvalue()


# ------------------------------------------------------------------------ measurement

def measure_allgather(shard_bytes: list, reps: int = 20, warmup: int = 3, group=None,
                      device=None) -> list:
    """Time ``all_gather_into_tensor`` of a ``shard_bytes`` payload per rank on the current
    process group, once per size; returns ``[(world, shard_bytes, seconds)]`` with seconds =
    mean per collective, max over ranks.  CUDA tensors (NCCL) are timed with CUDA events on
    the current stream, CPU tensors (gloo) with perf_counter; ranks are barrier-aligned."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    cuda = device is not None and torch.device(device).type == "cuda"
    out = []
    for nbytes in shard_bytes:
        words = max(1, -(-int(nbytes) // 4))
        inp = torch.zeros(words, dtype=torch.int32, device=device)
        gathered = torch.empty(world * words, dtype=torch.int32, device=device)
        for _ in range(warmup):
            dist.all_gather_into_tensor(gathered, inp, group=group)
        dist.barrier(group=group)
        if cuda:
            torch.cuda.synchronize()
            t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0.record()
            for _ in range(reps):
                dist.all_gather_into_tensor(gathered, inp, group=group)
            t1.record()
            torch.cuda.synchronize()
            sec = t0.elapsed_time(t1) / 1e3 / reps
        else:
            s0 = time.perf_counter()
            for _ in range(reps):
                dist.all_gather_into_tensor(gathered, inp, group=group)
            sec = (time.perf_counter() - s0) / reps
        t = torch.tensor([sec], dtype=torch.float64, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
        out.append((world, 4 * words, float(t.item())))
    return out


def fit_link(samples: list, source: str = "measured") -> LinkModel:
    """Least-squares fit of ``t / (N-1) = alpha + S / beta`` to ``[(N, S bytes, t)]``
    (N > 1).  A non-positive slope (latency-dominated samples) gives beta = inf."""
    pts = [(float(s), t / (n - 1)) for n, s, t in samples if n > 1]
    if len(pts) < 2:
        raise ValueError("fit_link needs at least two samples from a world of > 1 rank")
    mx = sum(p[0] for p in pts) / len(pts)
    my = sum(p[1] for p in pts) / len(pts)
    sxx = sum((p[0] - mx) ** 2 for p in pts)
    slope = sum((p[0] - mx) * (p[1] - my) for p in pts) / sxx if sxx > 0 else 0.0
    alpha = max(0.0, my - slope * mx)
    beta = 1.0 / slope if slope > 0 else math.inf
    return LinkModel(alpha, beta, source)
