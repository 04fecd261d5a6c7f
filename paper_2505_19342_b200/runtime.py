"""AstraRuntime — the B200 executor of the Astra lockstep SP forward.

Reference semantics: cluster.run_inference (cluster.py:224-308) with
_device_layer_compute (cluster.py:176-221) per device and layer.  Design:

* Layout.  Every device d holds, per image b, its T_d content rows followed by its
  class replica (if it owns one) — one flat fp32 "stack" [R, D] in HBM (the residual
  stream).  All devices of the plan that live on this GPU are laid out back to back
  ("virtual devices"); under torch.distributed each rank holds just its own shard.
* Per layer: VQ encode of the content rows (tcgen05 bf16x3 + exact fp64 re-rank) ->
  exchange of the packed codes (NCCL all-gather over NVLink; a no-op for virtual
  devices) -> LN1 -> fused Q|K|V GEMM over local rows -> attention whose K/V tile loader
  reads local keys from the projection buffer and remote keys straight out of the
  per-layer codebook K/V table by code (G = 1: LN1(C)·Wk, LN1(C)·Wv are exactly the rows
  the reference recomputes for every dequantized token) or from decoded K^/V^ (G > 1)
  -> Wo GEMM (+residual) -> LN2 -> W1 GEMM (+bias, erf-GELU) -> W2 GEMM (+bias,
  +residual).  Then the replica merge (device order), final LN and head GEMM.
* Precision.  "parity": every GEMM is split bf16x3 on tcgen05 (fp32-class; indices match
  the fp64 reference end to end), attention in fp32.  "fast": bf16 operands, fp32
  accumulate, fp32 residual stream; VQ encode stays exact in both modes.
* The whole forward is a fixed sequence of native launches on one stream, so it is
  captured once into a CUDA graph (``capture``) and replayed.
"""

from __future__ import annotations

import contextlib
import ctypes
import math
import os

import numpy as np
import torch

from . import _native, kernels
from .errors import IndexCorruptionError, LifecycleError, ShapeError
from .layout import sp_layout
from .model import LN_EPS, class_owner_ids
from .vq import DeviceCodebook, index_bits

BF16 = torch.bfloat16


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _p(t: torch.Tensor | None, elem_offset: int = 0) -> int | None:
    if t is None:
        return None
    return t.data_ptr() + elem_offset * t.element_size()


def _check_fp32(params) -> None:
    """The runtime keeps the reference's fp32 storage (tensor.py:26-31); an fp64 model would
    silently lose precision here, so it is rejected instead."""
    for name, t in params.named_tensors():
        dt = np.asarray(t.data).dtype
        if dt != np.float32:
            raise ShapeError(f"{name}: the B200 runtime stores fp32 parameters, got {dt}")
    for b in params.blocks:
        if b.codebook is not None:
            for c in b.codebook.centroids:
                if np.asarray(c).dtype != np.float32:
                    raise ShapeError("codebook centroids must be fp32 for the B200 runtime")


class TorchDistExchange:
    """Packed-index all-gather over torch.distributed (NCCL on NVLink/NVSwitch)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        # gloo (CPU tests, or several ranks sharing one GPU) moves host copies
        self.host_staged = dist.get_backend(group) == "gloo"

    def all_gather(self, out: torch.Tensor, inp: torch.Tensor) -> None:
        if not self.host_staged:
            self.dist.all_gather_into_tensor(out, inp, group=self.group)
            return
        parts = [torch.empty_like(inp, device="cpu") for _ in range(self.world)]
        self.dist.all_gather(parts, inp.cpu(), group=self.group)
        out.copy_(torch.cat(parts).view_as(out))

    def broadcast(self, t: torch.Tensor, src: int) -> None:
        if not self.host_staged:
            self.dist.broadcast(t, src=src, group=self.group)
            return
        h = t.cpu()
        self.dist.broadcast(h, src=src, group=self.group)
        t.copy_(h)


class LoopbackExchange:
    """Stand-in for one rank of an N-rank run on a single GPU (timing tool): every rank's slot
    of an all-gather receives this rank's own payload, a broadcast is a no-op.  The rank does
    exactly the work it would do under torchrun minus the NCCL transfer; its numerical
    results are not those of the real N-rank run."""

    def __init__(self, rank: int, world: int):
        self.rank, self.world = rank, world

    def all_gather(self, out: torch.Tensor, inp: torch.Tensor) -> None:
        out.view(self.world, -1).copy_(inp.reshape(1, -1).expand(self.world, -1))

    def broadcast(self, t: torch.Tensor, src: int) -> None:
        return None


class AstraRuntime:
    def __init__(self, params, plan, batch: int, mode: str = "classify",
                 cls_mode: str = "distributed", precision: str = "parity", comm=None,
                 device: torch.device | None = None, encode_at_one_device: bool = True,
                 require_codebooks: bool = True, sync_params: bool = True):
        if precision not in ("parity", "fast"):
            raise ValueError("precision must be 'parity' or 'fast'")
        if mode not in ("classify", "generate", "lm", "blocks"):
            raise ValueError(f"unknown runtime mode {mode!r}")
        if not torch.cuda.is_available():
            raise RuntimeError("AstraRuntime needs a CUDA device (no CPU fallback)")
        _native.load()
        cfg = params.config
        self.cfg, self.plan, self.B = cfg, plan, int(batch)
        self.mode, self.cls_mode, self.precision = mode, cls_mode, precision
        self.fast = precision == "fast"
        self.gelu_mode = 2 if self.fast else 1   # astra_gemm: 2 = bf16-class GELU polynomial
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        self.comm = comm
        self.sync_params = sync_params
        self.D, self.H, self.L = cfg.hidden, cfg.heads, cfg.layers
        self.dk = cfg.hidden // cfg.heads
        if self.dk > 128:
            raise ShapeError(f"head_dim {self.dk} unsupported (<= 128)")
        self.T, self.N = plan.tokens, plan.devices
        # K and G come from the codebooks actually attached (the reference's quantize reads
        # codebook.size / codebook.groups, vq.py:207-222 — e.g. exact_codebooks_from_reference
        # builds K = T tables, model.py:405-432); the config's values only size an
        # unquantized run.
        books = [b.codebook for b in params.blocks]
        if any(b is not None for b in books):
            if any(b is None for b in books):
                raise LifecycleError("codebooks must be initialized for all layers or none")
            sizes = {(b.size, b.groups, b.group_dim) for b in books}
            if len(sizes) != 1:
                raise ShapeError(f"all layers must share one codebook shape, got {sorted(sizes)}")
            self.K, self.G, gd = sizes.pop()
            if self.G * gd != cfg.hidden:
                raise ShapeError(f"codebook width {self.G * gd} != hidden {cfg.hidden}")
        else:
            self.G, self.K = cfg.groups, cfg.codebook_size
        self.bits = index_bits(self.K)
        _check_fp32(params)
        self.encode_at_one_device = encode_at_one_device
        self.require_codebooks = require_codebooks or plan.devices > 1
        self.capture_inputs = None   # setup hook: per-layer block inputs (codebook fitting)
        if comm is not None and comm.world != self.N:
            raise ShapeError("world size must equal plan.devices")
        self.local = list(range(self.N)) if comm is None else [comm.rank]
        self.owners = [] if cfg.causal else (class_owner_ids(plan, cls_mode)
                                             if plan.class_replication else [])
        self._build_layout()
        self._upload(params)
        self._alloc()
        # the VQ / exchange branch is on the critical path at N > 1: high stream priority
        self.side_stream = torch.cuda.Stream(device=self.device, priority=-1)
        self.overlap_vq = True   # False: strictly sequential launches (isolated kernel timing)
        self.qkv_after_vq = os.environ.get("ASTRA_QKV_PDL", "0") != "1"
        self._ev_fork, self._ev_join = torch.cuda.Event(), torch.cuda.Event()
        self.graph = None
        self.graphs = []
        self.x_slots = [self.x_in]
        self._slot = 0
        self.trace = None   # test hook: list collecting idx_all per layer
        self.profile = None  # bench hook: {op name: [(start_event, end_event), ...]}

    # ------------------------------------------------------------------ layout
    def _build_layout(self):
        lay = sp_layout(self.T, self.plan.ranges, self.B, self.local, self.owners)
        dev = self.device
        i32 = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.int32)).to(dev)  # noqa: E731
        self.row_base = lay.row_base
        self.R = lay.rows
        self.sizes = self.plan.shard_sizes()
        self.starts = [r[0] for r in self.plan.ranges]
        self.n_content = len(lay.content_rows)
        self.n_content_all = int(lay.gofs[-1])
        self.gofs = lay.gofs
        self.content_rows = i32(lay.content_rows)
        self.row_src, self.row_pos = i32(lay.row_src), i32(lay.row_pos)
        self.segs = i32(lay.segs.reshape(-1))
        self.n_segs = lay.segs.shape[0]
        self.key_map, self.key_pos = i32(lay.key_map), i32(lay.key_pos)
        self.n_keys = len(lay.key_map)
        self.rep_rows = i32(lay.rep_rows) if len(lay.rep_rows) else None
        self.max_nq = int(lay.segs[:, 1].max())
        self.has_remote = self.N > 1
        self.payload_bits = [self.B * s * self.G * self.bits for s in self.sizes]

    # ------------------------------------------------------------------ params
    def _to_dev(self, a) -> torch.Tensor:
        """Host fp32 array -> HBM.  Under torch.distributed every parameter is then broadcast
        from rank 0, so all ranks run bit-identical weights and codebooks whatever each
        process loaded (the reference's devices share one replicated model, cluster.py:259-265)."""
        arr = np.asarray(a.data if hasattr(a, "data") else a, np.float32)
        t = torch.from_numpy(np.array(arr, dtype=np.float32, copy=True)).to(self.device)
        if self.comm is not None and self.sync_params:
            self.comm.broadcast(t, src=0)
        return t

    def _wt(self, w_in_out: np.ndarray):
        """Reference weight [D_in, D_out] -> B operand [D_out, D_in] (hi[, lo])."""
        t = self._to_dev(w_in_out).t().contiguous()
        if self.fast:
            return t.to(BF16).contiguous(), None
        hi, lo = kernels.split_bf16(t)
        return hi.contiguous(), lo.contiguous()

    def _upload(self, params):
        dev = self.device
        f32 = self._to_dev
        self.layers = []
        for i, bp in enumerate(params.blocks):
            wqkv = np.concatenate([bp.wq.data, bp.wk.data, bp.wv.data], axis=1)
            lay = dict(
                wqkv=self._wt(wqkv), wo=self._wt(bp.wo.data), w1=self._wt(bp.w1.data),
                w2=self._wt(bp.w2.data), b1=f32(bp.b1), b2=f32(bp.b2),
                ln1_g=f32(bp.ln1_gain), ln1_b=f32(bp.ln1_bias),
                ln2_g=f32(bp.ln2_gain), ln2_b=f32(bp.ln2_bias))
            if bp.codebook is None:
                if self.require_codebooks:
                    raise ValueError(f"layer {i} has no codebook")
                lay["cb"] = None
            else:
                tables = np.stack([np.asarray(c, np.float32) for c in bp.codebook.centroids])
                lay["cb"] = DeviceCodebook(f32(tables), layer_id=i)
            self.layers.append(lay)
        self.pos = f32(params.pos)
        self.cls = f32(params.cls).reshape(-1) if params.cls is not None else None
        self.emb = f32(params.embedding) if params.embedding is not None else None
        self.final_g, self.final_b = f32(params.final_gain), f32(params.final_bias)
        self.head = self._wt(params.head.data)
        self.classes = params.head.data.shape[1]
        if self.has_remote and self.G == 1:
            self._build_kv_tables()
        del dev

    def _kv_rows(self, lay, x_f32: torch.Tensor, out: torch.Tensor, ln_hi, ln_lo):
        """K|V projection of fp32 rows: LN1 -> [Wk;Wv] GEMM (same kernels as the local path)."""
        m = x_f32.shape[0]
        D = self.D
        _native.call("astra_layernorm", x_f32.data_ptr(), m, D, x_f32.stride(0),
                     lay["ln1_g"].data_ptr(), lay["ln1_b"].data_ptr(), LN_EPS, None, 0,
                     ln_hi.data_ptr(), _p(ln_lo), D, _stream())
        self._kv_gemm(lay, m, out, ln_hi, ln_lo)

    def _kv_gemm(self, lay, m: int, out: torch.Tensor, ln_hi, ln_lo):
        """[Wk;Wv] projection of m LN1 rows (bf16 hi[, lo]) into out [m, 2D]."""
        D = self.D
        whi, wlo = lay["wqkv"]
        kernels.gemm(ln_hi[:m], whi[D:], a_lo=None if ln_lo is None else ln_lo[:m],
                     b_lo=None if wlo is None else wlo[D:],
                     out_f32=None if self.fast else out, out_hi=out if self.fast else None)

    def _build_kv_tables(self):
        """G = 1: per-layer codebook K/V tables [K, 2D] = (LN1(C) Wk | LN1(C) Wv)."""
        D, K = self.D, self.K
        ln_hi = torch.empty(K, D, dtype=BF16, device=self.device)
        ln_lo = None if self.fast else torch.empty_like(ln_hi)
        for lay in self.layers:
            c = lay["cb"].centroids[0]
            tab = torch.empty(K, 2 * D, dtype=BF16 if self.fast else torch.float32,
                              device=self.device)
            self._kv_rows(lay, c, tab, ln_hi, ln_lo)
            lay["kvtab"] = tab
        torch.cuda.current_stream().synchronize()

    # ----------------------------------------------------------------- buffers
    def _alloc(self):
        dev, R, D, B = self.device, self.R, self.D, self.B
        e = lambda *s, dt=torch.float32: torch.empty(*s, dtype=dt, device=dev)  # noqa: E731
        self.x_in = e(B * self.T, D)
        self.id_slots = [torch.zeros(B * self.T, dtype=torch.int32, device=dev)]
        self.X, self.Hres = e(R, D), e(R, D)
        self.ln_hi = e(R, D, dt=BF16)
        self.ln_lo = None if self.fast else e(R, D, dt=BF16)
        self.qkv = e(R, 3 * D, dt=BF16 if self.fast else torch.float32)
        self.o_hi = e(R, D, dt=BF16)
        self.o_lo = None if self.fast else e(R, D, dt=BF16)
        self.f_hi = e(R, 4 * D, dt=BF16)
        self.f_lo = None if self.fast else e(R, 4 * D, dt=BF16)
        self.idx_local = e(max(self.n_content, 1), self.G, dt=torch.int32)
        self.idx_all = self.idx_local if self.comm is None else e(self.n_content_all, self.G,
                                                                  dt=torch.int32)
        self.key_src = e(self.n_keys, dt=torch.int32)
        self.key_src.copy_(self.key_map)
        cb0 = self.layers[0]["cb"]
        # G = 1 and D a multiple of 128: LN1 also emits the bf16 split + row norms of the raw
        # stack, and the VQ distance GEMM consumes them directly (no separate split pass).
        self.presplit = (cb0 is not None and self.G == 1 and D in (512, 768, 1024))
        if self.presplit:
            self.xs_hi, self.xs_lo = e(R, D, dt=BF16), e(R, D, dt=BF16)
            self.xnorm = e(R)
            ws = int(_native.load().astra_vq_encode_split_workspace(R, self.K))
        else:
            self.xs_hi = self.xs_lo = self.xnorm = None
            ws = cb0.workspace_bytes(max(self.n_content, 1)) if cb0 else 1
        # zero-filled once: the fused VQ finalize's tile counters and re-rank list count are
        # self-cleaning after that (astra_vq_encode_split_ex)
        self.vq_ws = torch.zeros(max(ws, 1), dtype=torch.uint8, device=dev)
        # stack row -> token index (-1: replica rows), the inverse of content_rows
        rt = np.full(R, -1, dtype=np.int32)
        rt[self.content_rows.cpu().numpy()] = np.arange(self.n_content, dtype=np.int32)
        self.row_token = torch.from_numpy(rt).to(dev)
        # sticky device-side error flags: [0] a received code >= K (unpack / packed key map),
        # [1] a decode index out of range; read once per forward by check_errors()
        self.err_flags = torch.zeros(2, dtype=torch.int32, device=dev)
        self.vq_stats = torch.zeros(4, dtype=torch.int32, device=dev)
        self.collect_vq_stats = False   # exactness counters (re-rank rate); off on the hot path
        if self.comm is not None:
            wmax = (B * max(self.sizes) * self.G * self.bits + 31) // 32
            self.wmax = max(wmax, 1)
            self.words_local = torch.zeros(self.wmax, dtype=torch.int32, device=dev)
            self.words_all = torch.zeros(self.N * self.wmax, dtype=torch.int32, device=dev)
            self.unpack_err = self.err_flags[0:1]
            self.gofs_dev = torch.tensor(np.asarray(self.gofs, dtype=np.int32), device=dev)
        if self.has_remote and self.G > 1:
            n = self.n_content_all
            gd = D // self.G
            # decode fused into LN1 when the vector LN kernel covers the width (else decode ->
            # fp32 rows -> LN1); fused_decode = False is the A/B switch for the bench script
            self.fused_decode = D in (512, 768, 1024) and gd % 4 == 0
            self.xhat = None if self.fused_decode else e(n, D)
            self.hat_hi = e(n, D, dt=BF16)
            self.hat_lo = None if self.fast else e(n, D, dt=BF16)
            self.kvhat = e(n, 2 * D, dt=BF16 if self.fast else torch.float32)
            self.dec_err = self.err_flags[1:2]
        n_rep_local = 0 if self.rep_rows is None else self.rep_rows.numel()
        if self.mode == "generate":
            self._alloc_decode()
        if self.mode == "blocks":   # run_blocks: x0 is already embedded (no position add)
            self.pos_zero = torch.zeros_like(self.pos)
        if self.mode == "lm":       # lm_logits: final LN + head over every content row
            self.lm_ln_hi = e(R, D, dt=BF16)
            self.lm_ln_lo = None if self.fast else e(R, D, dt=BF16)
            self.lm_out = e(R, self.classes)
        if self.mode == "classify":
            self.reps_local = e(max(n_rep_local, 1), D)
            self.reps_all = e(len(self.owners) * B, D) if self.comm is not None else self.reps_local
            self.pooled = e(B, D)
            self.pool_hi = e(B, D, dt=BF16)
            self.pool_lo = None if self.fast else e(B, D, dt=BF16)
            self.logits = e(B, self.classes)

    # ------------------------------------------------------------ decode state
    def _alloc_decode(self):
        """Greedy generation on device N-1 (cluster.py:297-308): KV cache per layer holding
        its mixed view of the prompt (own rows full precision, remote rows K^/V^ of the
        received codes) plus every generated token, as DecodeState (model.py:324-334)."""
        dev, B, D, T = self.device, self.B, self.D, self.T
        self.dec_dev = self.N - 1
        self.decodes = self.dec_dev in self.local
        self.maxT = self.cfg.max_tokens
        i32 = lambda a: torch.tensor(np.asarray(a, dtype=np.int32), device=dev)  # noqa: E731
        sizes = self.sizes
        v = self.dec_dev
        # last content row of device N-1 for every image; its segment key range
        self.last_rows = i32([self.row_base[(v, b)] + sizes[v] - 1 for b in range(B)]) \
            if self.decodes else None
        if self.decodes:
            seg_idx = self.local.index(v) * B
            self.dec_k0 = int(self.segs.view(-1, 6)[seg_idx, 4].item())
        ebytes = 2 if self.fast else 4
        cdt = BF16 if self.fast else torch.float32
        self.ebytes = ebytes
        self.kv_cache = [torch.zeros(B * self.maxT, 2 * D, dtype=cdt, device=dev)
                         for _ in range(self.L)] if self.decodes else []
        self.dec_X = torch.empty(B, D, device=dev)
        self.dec_H = torch.empty(B, D, device=dev)
        self.dec_ln_hi = torch.empty(B, D, dtype=BF16, device=dev)
        self.dec_ln_lo = None if self.fast else torch.empty(B, D, dtype=BF16, device=dev)
        self.dec_qkv = torch.empty(B, 3 * D, dtype=cdt, device=dev)
        self.dec_o_hi = torch.empty(B, D, dtype=BF16, device=dev)
        self.dec_o_lo = None if self.fast else torch.empty(B, D, dtype=BF16, device=dev)
        self.dec_f_hi = torch.empty(B, 4 * D, dtype=BF16, device=dev)
        self.dec_f_lo = None if self.fast else torch.empty(B, 4 * D, dtype=BF16, device=dev)
        self.dec_logits = torch.empty(B, self.classes, device=dev)
        self.next_tok = torch.zeros(B, dtype=torch.int32, device=dev)
        self.first_out = torch.zeros(B, dtype=torch.int32, device=dev)
        self.dec_pos = torch.zeros(B, dtype=torch.int32, device=dev)
        self.dec_segs = torch.zeros(B * 6, dtype=torch.int32, device=dev)
        self.dec_key_src = i32([b * self.maxT + j for b in range(B) for j in range(self.maxT)])
        self.dec_key_pos = i32([j for _ in range(B) for j in range(self.maxT)])
        self.classes_out = None

    # ----------------------------------------------------------------- forward
    def _op(self, name: str):
        if self.profile is None:
            return contextlib.nullcontext()
        return self._timed(name)

    @contextlib.contextmanager
    def _timed(self, name: str):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        yield
        e.record()
        self.profile.setdefault(name, []).append((s, e))

    def _exchange(self, layer: int) -> bool:
        """Make every device's layer-`layer` codes visible to this GPU (cluster.py:276-279).
        Returns True when the key map was already resolved from the packed payload (G = 1)."""
        if self.comm is None:
            return False
        kernels.pack_indices(self.idx_local, self.bits, out=self.words_local)
        self.comm.all_gather(self.words_all, self.words_local)
        if self.G == 1 and self.trace is None:
            _native.call("astra_key_map_packed", self.key_map.data_ptr(), self.n_keys,
                         self.words_all.data_ptr(), self.wmax, self.bits, self.K,
                         self.gofs_dev.data_ptr(), self.N, self.key_src.data_ptr(),
                         self.unpack_err.data_ptr(), _stream())
            return True
        for e in range(self.N):
            cnt = self.B * self.sizes[e] * self.G
            kernels.unpack_indices(self.words_all[e * self.wmax:], cnt, self.bits, self.K,
                                   out=self.idx_all.view(-1)[int(self.gofs[e]) * self.G:],
                                   err=self.unpack_err)
        return False

    def _layer(self, l: int):
        lay = self.layers[l]
        D, R, s = self.D, self.R, _stream()
        cb = lay["cb"]
        if self.capture_inputs is not None:
            self.capture_inputs.append(self.X[self.content_rows.long()].clone())
        encode = cb is not None and (self.has_remote or self.encode_at_one_device)
        # 1. LN1 over the local stack (content + replica); with pre-split VQ it also writes the
        #    bf16 hi/lo split and norms of the raw rows from the same read
        split = self.presplit and encode
        with self._op("ln1"):
            _native.call("astra_layernorm_ex", self.X.data_ptr(), R, D, D,
                         lay["ln1_g"].data_ptr(), lay["ln1_b"].data_ptr(), LN_EPS, None, 0,
                         self.ln_hi.data_ptr(), _p(self.ln_lo), D,
                         _p(self.xs_hi) if split else None, _p(self.xs_lo) if split else None, D,
                         _p(self.xnorm) if split else None, s)
        # 2. VQ encode of this GPU's content tokens (cluster.py:272-275) and the exchange run on a
        #    side stream, overlapping the Q|K|V GEMM (the latency-bound finalize / re-rank
        #    kernels co-reside with the GEMM's CTAs).  They read X and the split LN1 wrote; the
        #    main stream joins before attention (N > 1: the remote keys) or before W2 (N = 1:
        #    W2 overwrites X).
        main = torch.cuda.current_stream()
        side_work = (encode or self.has_remote) and self.overlap_vq
        if side_work:
            self._ev_fork.record(main)
            self.side_stream.wait_event(self._ev_fork)
        side_ctx = torch.cuda.stream(self.side_stream) if side_work else contextlib.nullcontext()
        with side_ctx:
            remote = self._encode_exchange(l, lay, cb, encode, split)
            if side_work:
                self._ev_join.record(self.side_stream)
        if side_work and self.trace is not None:
            main.wait_event(self._ev_join)   # test hook reads the codes now
            self.trace.append(self.idx_all.clone())
        elif self.trace is not None:
            self.trace.append(self.idx_all.clone())
        # 4. fused Q|K|V projection.  With remote keys the VQ chain, not this GEMM, gates the
        #    attention: launched without programmatic early start, the GEMM's persistent CTAs do
        #    not occupy the SMs before LN1 ends, and the (high-priority) VQ GEMM goes first.
        whi, wlo = lay["wqkv"]
        late = side_work and self.has_remote and self.qkv_after_vq
        prev = _native.load().astra_pdl_override(0) if late else None
        try:
            with self._op("gemm_qkv"):
                kernels.gemm(self.ln_hi, whi, a_lo=self.ln_lo, b_lo=wlo,
                             out_f32=None if self.fast else self.qkv,
                             out_hi=self.qkv if self.fast else None)
        finally:
            if late:
                _native.load().astra_pdl_override(prev)
        joined = not side_work or self.trace is not None
        self._layer_rest(l, lay, remote, join_before_attn=not joined and self.has_remote,
                         join_before_w2=not joined and not self.has_remote)

    def _encode_exchange(self, l, lay, cb, encode, split):
        """VQ encode + exchange + remote K/V view (on the current stream); returns the remote
        K/V buffer for the attention kernel."""
        D, R, s = self.D, self.R, _stream()
        if encode:
            with self._op("vq_encode"):
                if split:
                    _native.call("astra_vq_encode_split_ex", ctypes.byref(cb.struct),
                                 self.X.data_ptr(), D, self.xs_hi.data_ptr(),
                                 self.xs_lo.data_ptr(), D, self.xnorm.data_ptr(), R,
                                 self.content_rows.data_ptr(), self.n_content,
                                 self.row_token.data_ptr(), self.idx_local.data_ptr(),
                                 self.vq_stats.data_ptr() if self.collect_vq_stats else None,
                                 self.vq_ws.data_ptr(), self.vq_ws.numel(), s)
                else:
                    cb.encode(self.X, out=self.idx_local, rows=self.content_rows,
                              workspace=self.vq_ws,
                              stats=self.vq_stats if self.collect_vq_stats else None)
        # 2. exchange + remote K/V view
        if self.has_remote:
            with self._op("exchange"):
                resolved = self._exchange(l)
            if self.G == 1:
                if not resolved:
                    _native.call("astra_key_map", self.key_map.data_ptr(), self.n_keys,
                                 self.idx_all.data_ptr(), self.key_src.data_ptr(), s)
                remote = lay["kvtab"]
            else:
                with self._op("decode_ln"):
                    if self.fused_decode:
                        # decode fused into LN1: received codes -> LN1(C[idx]) as the K|V
                        # projection's bf16 operand, no fp32 decoded rows in HBM
                        _native.call("astra_vq_decode_layernorm", ctypes.byref(cb.struct),
                                     self.idx_all.data_ptr(), self.n_content_all,
                                     lay["ln1_g"].data_ptr(), lay["ln1_b"].data_ptr(), LN_EPS,
                                     self.hat_hi.data_ptr(), _p(self.hat_lo), D, self.dec_err.data_ptr(), s)
                    else:
                        cb.decode(self.idx_all, out=self.xhat, err=self.dec_err)
                        _native.call("astra_layernorm", self.xhat.data_ptr(), self.n_content_all, D, D,
                                     lay["ln1_g"].data_ptr(), lay["ln1_b"].data_ptr(), LN_EPS, None, 0,
                                     self.hat_hi.data_ptr(), _p(self.hat_lo), D, s)
                with self._op("gemm_kv"):
                    self._kv_gemm(lay, self.n_content_all, self.kvhat, self.hat_hi, self.hat_lo)
                remote = self.kvhat
        else:
            remote = self.qkv
        return remote

    def _layer_rest(self, l, lay, remote, join_before_attn: bool, join_before_w2: bool):
        D, R, s = self.D, self.R, _stream()
        if join_before_attn:
            torch.cuda.current_stream().wait_event(self._ev_join)   # remote keys resolved
        if self.mode == "generate" and self.decodes:
            # DecodeState capture (cluster.py:285-288): device N-1's K|V view of the prompt
            e = self.ebytes
            with self._op("kv_capture"):
                _native.call("astra_gather_kv", self.key_src.data_ptr() + 4 * self.dec_k0,
                             self.B * self.T, self.T, self.maxT, _p(self.qkv, D),
                             _p(self.qkv, 2 * D), 3 * D * e, _p(remote, 0), _p(remote, D),
                             remote.stride(0) * e, D * e, self.kv_cache[l].data_ptr(), 2 * D * e,
                             s)
        # 5. mixed-precision attention
        ld_r = remote.stride(0)
        with self._op("attention"):
            _native.call("astra_attention", self.qkv.data_ptr(), 3 * D, _p(self.qkv, D),
                     _p(self.qkv, 2 * D), 3 * D, _p(remote, 0 if remote is self.qkv else 0),
                     _p(remote, D), ld_r, self.key_src.data_ptr(), self.key_pos.data_ptr(),
                     self.segs.data_ptr(), self.n_segs, self.max_nq, self.H, self.dk,
                     2 if self.cfg.causal else 0,   # causal layouts hold prefix keys (layout.py)
                     int(self.fast), float(np.float32(1.0 / math.sqrt(self.dk))),
                     None, self.o_hi.data_ptr(), _p(self.o_lo), D, R, R, remote.shape[0], s)
        # 6. h = stack + attn Wo
        whi, wlo = lay["wo"]
        with self._op("gemm_wo"):
            kernels.gemm(self.o_hi, whi, a_lo=self.o_lo, b_lo=wlo, residual=self.X,
                         out_f32=self.Hres)
        # 7. LN2 -> W1 (+b1, GELU) -> W2 (+b2, +h)
        with self._op("ln2"):
            _native.call("astra_layernorm", self.Hres.data_ptr(), R, D, D, lay["ln2_g"].data_ptr(),
                     lay["ln2_b"].data_ptr(), LN_EPS, None, 0, self.ln_hi.data_ptr(),
                     _p(self.ln_lo), D, s)
        whi, wlo = lay["w1"]
        with self._op("gemm_w1"):
            kernels.gemm(self.ln_hi, whi, a_lo=self.ln_lo, b_lo=wlo, bias=lay["b1"], gelu=self.gelu_mode,
                         out_hi=self.f_hi, out_lo=self.f_lo)
        whi, wlo = lay["w2"]
        if join_before_w2:
            torch.cuda.current_stream().wait_event(self._ev_join)   # VQ reads of X are done
        with self._op("gemm_w2"):
            kernels.gemm(self.f_hi, whi, a_lo=self.f_lo, b_lo=wlo, bias=lay["b2"],
                         residual=self.Hres, out_f32=self.X)

    def _embed(self):
        # classify: x + pos (model.py:275-280); generate: embedding[ids] + pos (model.py:283-288)
        if self.mode in ("generate", "lm"):
            _native.call("astra_embed_tokens", self.emb.data_ptr(), self.pos.data_ptr(),
                         self.id_slots[self._slot].data_ptr(), self.row_src.data_ptr(),
                         self.row_pos.data_ptr(), self.R, self.D, self.X.data_ptr(), _stream())
            return
        x_in = self.x_slots[self._slot]
        pos = self.pos_zero if self.mode == "blocks" else self.pos
        _native.call("astra_embed_stack", x_in.data_ptr(), pos.data_ptr(),
                     _p(self.cls), self.row_src.data_ptr(), self.row_pos.data_ptr(), self.R,
                     self.D, self.X.data_ptr(), _stream())

    def _classify_tail(self):
        D, B, s = self.D, self.B, _stream()
        n_loc = self.rep_rows.numel() if self.rep_rows is not None else 0
        if n_loc:
            _native.call("astra_gather_rows", self.X.data_ptr(), D, self.rep_rows.data_ptr(),
                         n_loc, D, self.reps_local.data_ptr(), D, s)
        if self.comm is not None:
            self._gather_replicas()
        _native.call("astra_replica_mean", self.reps_all.data_ptr(), len(self.owners), B, D,
                     self.pooled.data_ptr(), s)
        _native.call("astra_layernorm", self.pooled.data_ptr(), B, D, D, self.final_g.data_ptr(),
                     self.final_b.data_ptr(), LN_EPS, None, 0, self.pool_hi.data_ptr(),
                     _p(self.pool_lo), D, s)
        whi, wlo = self.head
        kernels.gemm(self.pool_hi, whi, a_lo=self.pool_lo, b_lo=wlo, out_f32=self.logits)

    def _gather_replicas(self):
        """Replica merge across ranks (cluster.py:290-292): all-gather [B, D] per owner."""
        B, D = self.B, self.D
        buf = getattr(self, "_rep_gather", None)
        if buf is None:
            self._rep_gather = buf = torch.zeros(self.N * B, D, device=self.device)
            self._rep_send = torch.zeros(B, D, device=self.device)
        if self.rep_rows is not None:
            self._rep_send.copy_(self.reps_local[:B])
        else:
            self._rep_send.zero_()
        self.comm.all_gather(buf, self._rep_send)
        for i, e in enumerate(self.owners):
            self.reps_all[i * B:(i + 1) * B].copy_(buf[e * B:(e + 1) * B])

    def forward(self):
        """Run the forward on the already-staged input ``self.x_in``; logits in ``self.logits``."""
        with self._op("embed"):
            self._embed()
        for l in range(self.L):
            self._layer(l)
        if self.mode == "classify":
            with self._op("tail"):
                self._classify_tail()
            return self.logits
        if self.mode == "lm":
            self._lm_tail()
            return self.lm_out
        if self.mode == "generate" and self.decodes:
            self._first_token()
            return self.first_out
        return None

    def _first_token(self):
        """End of the prefill (cluster.py:299-302): greedy first token of every sequence from
        the decoding device's last row -> first_out / next_tok."""
        _native.call("astra_gather_rows", self.X.data_ptr(), self.D, self.last_rows.data_ptr(),
                     self.B, self.D, self.dec_X.data_ptr(), self.D, _stream())
        self._head_argmax(self.dec_X, self.first_out, 1, first=True)

    def _lm_tail(self):
        """lm_logits (model.py:305-313): final LN and head over every content row (causal
        stacks hold no replicas)."""
        D, R, s = self.D, self.R, _stream()
        _native.call("astra_layernorm", self.X.data_ptr(), R, D, D, self.final_g.data_ptr(),
                     self.final_b.data_ptr(), LN_EPS, None, 0, self.lm_ln_hi.data_ptr(),
                     _p(self.lm_ln_lo), D, s)
        whi, wlo = self.head
        kernels.gemm(self.lm_ln_hi, whi, a_lo=self.lm_ln_lo, b_lo=wlo, out_f32=self.lm_out)

    # -------------------------------------------------------------- CUDA graph
    def _add_slots(self, slots: int):
        while len(self.x_slots) < slots:
            self.x_slots.append(torch.empty_like(self.x_in))
        while len(self.id_slots) < slots:
            self.id_slots.append(torch.zeros_like(self.id_slots[0]))

    def capture(self, warmup: int = 1, slots: int = 1):
        """Record ``forward`` (fixed buffers, fixed launch sequence) into CUDA graphs, one per
        input slot (two slots let the next batch's host->device copy overlap this forward)."""
        self._add_slots(slots)
        for _ in range(warmup):
            self.forward()
        torch.cuda.synchronize()
        self.graphs = []
        for slot in range(len(self.x_slots)):
            self._slot = slot
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                self.forward()
            self.graphs.append(g)
        self._slot = 0
        self.graph = self.graphs[0]
        return self.graph

    def run(self, slot: int = 0):
        if self.graph is not None:
            self.graphs[slot].replay()
        else:
            self._slot = slot
            self.forward()
            self._slot = 0
        return getattr(self, "logits", None)

    def _serve(self, batches, out, stage, result):
        """Double-buffered serving loop: the host->device copy of batch i+1 (``stage``) runs on
        a copy stream while batch i's forward runs; each batch's ``result`` is copied back, and
        the host waits for it only after batch i+1's forward has been enqueued."""
        if len(self.x_slots) < 2:
            try:
                self.capture(slots=2)
            except RuntimeError:   # e.g. a collective that cannot be graph-captured: eager
                torch.cuda.synchronize()
                self.graph, self.graphs = None, []
                self._add_slots(2)
        main = torch.cuda.current_stream()
        copy = getattr(self, "_copy_stream", None) or torch.cuda.Stream(device=self.device)
        self._copy_stream = copy
        copied = [torch.cuda.Event() for _ in range(2)]
        done = [torch.cuda.Event() for _ in range(2)]
        results = []
        n = len(batches)

        def h2d(i):
            slot = i % 2
            with torch.cuda.stream(copy):
                if i >= 2:
                    copy.wait_event(done[slot])
                stage(slot, batches[i])
                copied[slot].record(copy)

        if n:
            h2d(0)
        fetched = [torch.cuda.Event() for _ in range(2)]
        pending = None   # (host buffer, event) of the previous batch's result
        for i in range(n):
            slot = i % 2
            main.wait_event(copied[slot])
            self.run(slot)
            done[slot].record(main)
            if i + 1 < n:
                h2d(i + 1)
            host = out[i] if out is not None else torch.empty(result.shape, dtype=result.dtype,
                                                              pin_memory=True)
            host.copy_(result, non_blocking=True)   # stream order: before batch i+1 overwrites it
            fetched[slot].record(main)
            # one batch stays queued behind the host: wait for the PREVIOUS batch's result only,
            # so the next forward is already enqueued while the host takes this one
            if pending is not None:
                pending[1].synchronize()
                results.append(pending[0])
            pending = (host, fetched[slot])
        if pending is not None:
            pending[1].synchronize()
            results.append(pending[0])
        self.check_errors()
        return results

    def classify_stream(self, batches, out=None):
        """Serve host batches ([B, T, D] fp32, pinned; under torchrun this rank's token shard
        [B, T_d, D]) -> host logits per batch."""
        start, stop = ((0, self.T) if self.comm is None else self.plan.ranges[self.comm.rank])

        def stage(slot, src):
            xv = self.x_slots[slot].view(self.B, self.T, self.D)
            if self.comm is None:
                xv.copy_(src, non_blocking=True)
            else:  # only this rank's token shard crosses PCIe
                xv[:, start:stop].copy_(src, non_blocking=True)

        return self._serve(batches, out, stage, self.logits)

    def prefill_stream(self, batches, out=None):
        """Serve host token-id batches ([B, T] int32, pinned) through the SP causal prefill ->
        the first greedy token of every sequence (host int32 [B]) per batch."""
        if self.mode != "generate":
            raise ValueError("runtime was not built for generate mode")

        def stage(slot, src):
            self.id_slots[slot].view(self.B, self.T).copy_(src, non_blocking=True)

        return self._serve(batches, out, stage, self.first_out)

    # ------------------------------------------------------------------ host API
    def stage_input(self, xs):
        """Copy inputs [B, T, D] (host NumPy/pinned tensor or device tensor) into HBM."""
        if isinstance(xs, np.ndarray):
            xs = torch.from_numpy(np.ascontiguousarray(xs, dtype=np.float32))
        if xs.shape != (self.B, self.T, self.D):
            raise ShapeError(f"expected inputs [{self.B}, {self.T}, {self.D}], got {tuple(xs.shape)}")
        self.x_in.view(self.B, self.T, self.D).copy_(xs, non_blocking=True)

    def check_errors(self) -> None:
        """Raise IndexCorruptionError if any received / decoded VQ code of the forwards since
        the last check was outside [0, K) — the reference's dequantize check (vq.py:229-231).
        One 8-byte device->host read; the flags are cleared after a raise."""
        f = self.err_flags.cpu().numpy()
        if f.any():
            self.err_flags.zero_()
            where = "in the exchanged payload" if f[0] else "at decode"
            raise IndexCorruptionError(f"VQ index outside [0, {self.K}) {where}")

    def record_ledger(self, ledger):
        if ledger is None or self.N <= 1:
            return
        for l in range(self.L):
            ledger.record_exchange(l, self.payload_bits)

    # ---------------------------------------------------------------- generate
    def _gemm_rows(self, w, a_hi, a_lo, **kw):
        whi, wlo = w
        kernels.gemm(a_hi, whi, a_lo=a_lo, b_lo=wlo, **kw)

    def _head_argmax(self, x_rows: torch.Tensor, out: torch.Tensor, steps: int, first: bool):
        """final LN -> head -> greedy argmax (lowest id on ties, cluster.py:299-302)."""
        B, D, s = self.B, self.D, _stream()
        _native.call("astra_layernorm", x_rows.data_ptr(), B, D, D, self.final_g.data_ptr(),
                     self.final_b.data_ptr(), LN_EPS, None, 0, self.dec_ln_hi.data_ptr(),
                     _p(self.dec_ln_lo), D, s)
        self._gemm_rows(self.head, self.dec_ln_hi, self.dec_ln_lo, out_f32=self.dec_logits)
        _native.call("astra_argmax_rows", self.dec_logits.data_ptr(), B, self.classes,
                     self.classes, out.data_ptr(), steps, None if first else self.dec_pos.data_ptr(),
                     self.T - 1, self.next_tok.data_ptr(), s)

    def _decode_step(self, out: torch.Tensor, steps: int):
        """One greedy step for every image (model.py:337-358) on the decoding device."""
        B, D, s = self.B, self.D, _stream()
        e = self.ebytes
        X, H = self.dec_X, self.dec_H
        _native.call("astra_embed_stack", self.emb.data_ptr(), self.pos.data_ptr(), None,
                     self.next_tok.data_ptr(), self.dec_pos.data_ptr(), B, D, X.data_ptr(), s)
        scale = float(np.float32(1.0 / math.sqrt(self.dk)))
        for l, lay in enumerate(self.layers):
            cache = self.kv_cache[l]
            _native.call("astra_layernorm", X.data_ptr(), B, D, D, lay["ln1_g"].data_ptr(),
                         lay["ln1_b"].data_ptr(), LN_EPS, None, 0, self.dec_ln_hi.data_ptr(),
                         _p(self.dec_ln_lo), D, s)
            self._gemm_rows(lay["wqkv"], self.dec_ln_hi, self.dec_ln_lo,
                            out_f32=None if self.fast else self.dec_qkv,
                            out_hi=self.dec_qkv if self.fast else None)
            _native.call("astra_append_kv", _p(self.dec_qkv, D), _p(self.dec_qkv, 2 * D),
                         3 * D * e, B, self.dec_pos.data_ptr(), self.maxT, D * e,
                         cache.data_ptr(), 2 * D * e, s)
            _native.call("astra_attention", self.dec_qkv.data_ptr(), 3 * D, cache.data_ptr(),
                         _p(cache, D), 2 * D, cache.data_ptr(), _p(cache, D), 2 * D,
                         self.dec_key_src.data_ptr(), self.dec_key_pos.data_ptr(),
                         self.dec_segs.data_ptr(), B, 1, self.H, self.dk, 0, int(self.fast),
                         scale, None, self.dec_o_hi.data_ptr(), _p(self.dec_o_lo), D, B,
                         cache.shape[0], cache.shape[0], s)
            self._gemm_rows(lay["wo"], self.dec_o_hi, self.dec_o_lo, residual=X, out_f32=H)
            _native.call("astra_layernorm", H.data_ptr(), B, D, D, lay["ln2_g"].data_ptr(),
                         lay["ln2_b"].data_ptr(), LN_EPS, None, 0, self.dec_ln_hi.data_ptr(),
                         _p(self.dec_ln_lo), D, s)
            self._gemm_rows(lay["w1"], self.dec_ln_hi, self.dec_ln_lo, bias=lay["b1"], gelu=self.gelu_mode,
                            out_hi=self.dec_f_hi, out_lo=self.dec_f_lo)
            self._gemm_rows(lay["w2"], self.dec_f_hi, self.dec_f_lo, bias=lay["b2"], residual=H,
                            out_f32=X)
        self._head_argmax(X, out, steps, first=False)
        _native.call("astra_decode_advance", self.dec_pos.data_ptr(), self.dec_segs.data_ptr(), B, s)

    def set_ids(self, ids, slot: int = 0) -> None:
        """Stage token ids [B, T] (embedding[ids] + pos, model.py:283-288) into HBM."""
        B, T = self.B, self.T
        ids = np.asarray(ids, dtype=np.int64).reshape(B, T)
        if ids.size and (ids.min() < 0 or ids.max() >= self.emb.shape[0]):
            raise ShapeError("gather_rows: id out of range")
        self.id_slots[slot].copy_(torch.from_numpy(ids.astype(np.int32).reshape(-1)))

    def lm_logits(self, ids) -> np.ndarray:
        """[B, T, vocab] next-token logits of every position (mode "lm")."""
        if self.mode != "lm":
            raise ValueError("runtime was not built for lm mode")
        self.set_ids(ids)
        self.forward()
        out = self.codes_by_image(self.lm_out[self.content_rows.long()], self.classes)
        self.check_errors()
        return out

    def stack_by_image(self):
        """After a forward: content rows [B, T, D] in global token order and the class replicas
        [B, n_owners, D] in owner order (run_blocks' (content, replicas), model.py:198-265)."""
        content = self.codes_by_image(self.X[self.content_rows.long()], self.D)
        reps = None
        if self.rep_rows is not None and self.comm is None:
            r = self.X[self.rep_rows.long()].cpu().numpy()       # (v, b) order
            reps = r.reshape(len(self.owners), self.B, self.D).transpose(1, 0, 2).copy()
        return content, reps

    def project_kv(self, l: int, rows: torch.Tensor) -> np.ndarray:
        """LN1(rows) @ [Wk | Wv] of layer l as fp32 [m, 2D] — the K/V the reference derives
        from a layer input (cluster.py:196-198) — for run_blocks' on_layer observers."""
        m = rows.shape[0]
        rows = rows.float().contiguous()
        hi = torch.empty(m, self.D, dtype=BF16, device=self.device)
        lo = None if self.fast else torch.empty_like(hi)
        out = torch.empty(m, 2 * self.D, dtype=BF16 if self.fast else torch.float32,
                          device=self.device)
        self._kv_rows(self.layers[l], rows, out, hi, lo)
        return out.float().cpu().numpy()

    def generate(self, ids, steps: int, ledger=None) -> np.ndarray:
        """Sequence-parallel causal prefill, then greedy decode on device N-1
        (cluster.py:243-308).  ids: [B, T] prompt token ids -> [B, steps] generated ids."""
        if self.mode != "generate":
            raise ValueError("runtime was not built for generate mode")
        B, dev = self.B, self.device
        T = self.T
        self.set_ids(ids)
        out = torch.zeros(B, max(steps, 1), dtype=torch.int32, device=dev)
        self.run()
        self.record_ledger(ledger)
        if self.decodes and steps > 0:
            out[:, 0].copy_(self.first_out)
            segs = np.array([[b, 1, T, 1, b * self.maxT, T + 1] for b in range(B)], np.int32)
            self.dec_segs.copy_(torch.from_numpy(segs.reshape(-1)))
            self.dec_pos.fill_(T)
            for _ in range(1, steps):
                self._decode_step(out, steps)
        if self.comm is not None:
            self.comm.broadcast(out, src=self.dec_dev)
        res = out[:, :steps].cpu().numpy()
        self.check_errors()
        return res

    def classify_numpy(self, xs: np.ndarray, ledger=None) -> np.ndarray:
        self.stage_input(xs)
        out = self.run().cpu().numpy().copy()
        self.check_errors()
        self.record_ledger(ledger)
        return out

    def indices_after_layer(self):
        return self.idx_all

    def codes_by_image(self, idx: torch.Tensor, width: int | None = None) -> np.ndarray:
        """Per-content-row data of every device in global-content order (e, b, r) -> [B, T, width]
        in global token order per image — for codes (width G, what the reference's per-device
        quantize calls produce in device order, cluster.py:272-275) or captured rows (width D)."""
        width = self.G if width is None else width
        a = idx.reshape(-1, width).cpu().numpy()
        out = np.empty((self.B, self.T, width), a.dtype)
        for e in range(self.N):
            blk = a[int(self.gofs[e]):int(self.gofs[e + 1])].reshape(self.B, self.sizes[e], width)
            out[:, self.starts[e]:self.starts[e] + self.sizes[e]] = blk
        return out
