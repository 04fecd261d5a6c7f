"""Model configuration and parameters — drop-in for seqvq.model (model.py:31-169, 435-482).

Parameters are generated exactly like the reference (named PCG64 streams,
rng.py:32-37), so a given (config, seed) yields bit-identical fp32 weights on
both sides.  Arrays live on the host as NumPy; ``runtime.AstraRuntime``
uploads them to HBM once.
"""

from __future__ import annotations

import hashlib
import struct
from dataclasses import dataclass

import numpy as np

from .errors import LifecycleError, ShapeError
from .vq import Codebook, load_codebook, save_codebook

CHECKPOINT_MAGIC = b"ASTM"
LN_EPS = 1e-5


def _stable_hash(name) -> int:
    """rng.py:24-29"""
    if isinstance(name, (int, np.integer)):
        return int(name) & 0xFFFFFFFFFFFFFFFF
    return int.from_bytes(hashlib.sha256(str(name).encode("utf-8")).digest()[:8], "little")


def generator(seed: int, *names) -> np.random.Generator:
    """rng.generator (rng.py:32-37): PCG64 over SeedSequence([seed, H(name)...])."""
    if not isinstance(seed, (int, np.integer)):
        raise TypeError(f"seed must be an integer, got {type(seed).__name__}")
    entropy = [int(seed) & 0xFFFFFFFFFFFFFFFF] + [_stable_hash(n) for n in names]
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence(entropy)))


class Tensor:
    """Immutable array holder with the reference's ``.data`` accessor (tensor.py:21-57)."""

    __slots__ = ("data",)

    def __init__(self, data, dtype=None):
        arr = np.array(data, copy=True)
        if dtype is not None:
            arr = arr.astype(dtype)
        elif arr.dtype not in (np.float32, np.float64):
            arr = arr.astype(np.float32)
        arr.flags.writeable = False
        self.data = arr

    @property
    def shape(self):
        return self.data.shape

    @property
    def dtype(self):
        return self.data.dtype


@dataclass(frozen=True)
class ModelConfig:
    """model.py:31-56 (same fields, defaults and validation)."""

    layers: int
    hidden: int
    heads: int
    vocab_or_classes: int
    max_tokens: int
    causal: bool
    mlp_expansion: int = 4
    codebook_size: int = 16
    groups: int = 1

    def __post_init__(self):
        if self.layers < 1:
            raise ValueError("need at least one layer")
        if self.hidden % self.heads != 0:
            raise ShapeError(f"hidden {self.hidden} not divisible by {self.heads} heads")
        if self.hidden % self.groups != 0:
            raise ShapeError(f"hidden {self.hidden} not divisible by {self.groups} groups")
        if self.vocab_or_classes < 2:
            raise ValueError("need at least two classes / vocabulary entries")

    @property
    def class_token(self) -> bool:
        return not self.causal


@dataclass
class BlockParams:
    """model.py:59-77"""

    wq: Tensor
    wk: Tensor
    wv: Tensor
    wo: Tensor
    w1: Tensor
    b1: Tensor
    w2: Tensor
    b2: Tensor
    ln1_gain: Tensor
    ln1_bias: Tensor
    ln2_gain: Tensor
    ln2_bias: Tensor
    codebook: Codebook | None = None

    TENSOR_FIELDS = ("wq", "wk", "wv", "wo", "w1", "b1", "w2", "b2",
                     "ln1_gain", "ln1_bias", "ln2_gain", "ln2_bias")


@dataclass
class ModelParams:
    """model.py:80-123"""

    config: ModelConfig
    pos: Tensor
    blocks: list
    final_gain: Tensor
    final_bias: Tensor
    head: Tensor
    embedding: Tensor | None = None
    cls: Tensor | None = None

    def named_tensors(self):
        out = []
        if self.embedding is not None:
            out.append(("embedding", self.embedding))
        out.append(("pos", self.pos))
        if self.cls is not None:
            out.append(("cls", self.cls))
        for i, b in enumerate(self.blocks):
            for f in BlockParams.TENSOR_FIELDS:
                out.append((f"block{i}.{f}", getattr(b, f)))
        out.extend([("final_gain", self.final_gain), ("final_bias", self.final_bias),
                    ("head", self.head)])
        return out

    def assign(self, name: str, data: np.ndarray) -> None:
        if name.startswith("block"):
            idx, f = name.split(".", 1)
            setattr(self.blocks[int(idx[5:])], f, Tensor(data))
        else:
            setattr(self, name, Tensor(data))


def init_params(config: ModelConfig, seed: int, dtype=np.float32,
                init_scale: float = 0.02) -> ModelParams:
    """model.py:126-160: Gaussian init scaled by init_scale; layer norms at identity."""
    d = config.hidden
    m = d * config.mlp_expansion

    def w(name, shape, scl=init_scale):
        return Tensor(generator(seed, "init", name).normal(size=shape) * scl, dtype=dtype)

    def ones(shape):
        return Tensor(np.ones(shape), dtype=dtype)

    def zeros(shape):
        return Tensor(np.zeros(shape), dtype=dtype)

    blocks = []
    for i in range(config.layers):
        blocks.append(BlockParams(
            wq=w(f"b{i}.wq", (d, d)), wk=w(f"b{i}.wk", (d, d)),
            wv=w(f"b{i}.wv", (d, d)), wo=w(f"b{i}.wo", (d, d)),
            w1=w(f"b{i}.w1", (d, m)), b1=zeros((m,)),
            w2=w(f"b{i}.w2", (m, d)), b2=zeros((d,)),
            ln1_gain=ones((d,)), ln1_bias=zeros((d,)),
            ln2_gain=ones((d,)), ln2_bias=zeros((d,)),
        ))
    return ModelParams(
        config=config,
        embedding=w("embedding", (config.vocab_or_classes, d)) if config.causal else None,
        pos=w("pos", (config.max_tokens, d), 0.01),
        cls=w("cls", (1, d)) if config.class_token else None,
        blocks=blocks,
        final_gain=ones((d,)), final_bias=zeros((d,)),
        head=w("head", (d, config.vocab_or_classes)),
    )


def class_owner_ids(plan, cls_mode: str) -> list[int]:
    """Devices holding a class-token replica (model.py:163-169)."""
    if cls_mode == "distributed":
        return list(range(plan.devices))
    if cls_mode == "single":
        return [0]
    raise ValueError(f"unknown cls_mode {cls_mode!r}")


def save_checkpoint(params: ModelParams) -> bytes:
    """ASTM container (model.py:435-451): magic, version, config, fp32 LE tensors, codebooks."""
    cfg = params.config
    out = [CHECKPOINT_MAGIC, struct.pack("<10I", 1, cfg.layers, cfg.hidden, cfg.heads,
                                         cfg.vocab_or_classes, cfg.max_tokens, int(cfg.causal),
                                         cfg.mlp_expansion, cfg.codebook_size, cfg.groups)]
    for _, t in params.named_tensors():
        out.append(np.ascontiguousarray(t.data, dtype="<f4").tobytes())
    books = [b.codebook for b in params.blocks if b.codebook is not None]
    out.append(struct.pack("<I", len(books)))
    for cb in books:
        blob = save_codebook(cb)
        out.append(struct.pack("<I", len(blob)))
        out.append(blob)
    return b"".join(out)


def load_checkpoint(blob: bytes) -> ModelParams:
    """Inverse of save_checkpoint (model.py:454-482), same validation."""
    if blob[:4] != CHECKPOINT_MAGIC:
        raise ValueError("not a model checkpoint (bad magic)")
    fields = struct.unpack("<10I", blob[4:44])
    if fields[0] != 1:
        raise ValueError(f"unsupported checkpoint version {fields[0]}")
    cfg = ModelConfig(layers=fields[1], hidden=fields[2], heads=fields[3],
                      vocab_or_classes=fields[4], max_tokens=fields[5], causal=bool(fields[6]),
                      mlp_expansion=fields[7], codebook_size=fields[8], groups=fields[9])
    d, m = cfg.hidden, cfg.hidden * cfg.mlp_expansion
    shapes = []
    if cfg.causal:
        shapes.append(("embedding", (cfg.vocab_or_classes, d)))
    shapes.append(("pos", (cfg.max_tokens, d)))
    if not cfg.causal:
        shapes.append(("cls", (1, d)))
    blk = dict(wq=(d, d), wk=(d, d), wv=(d, d), wo=(d, d), w1=(d, m), b1=(m,), w2=(m, d), b2=(d,),
               ln1_gain=(d,), ln1_bias=(d,), ln2_gain=(d,), ln2_bias=(d,))
    for i in range(cfg.layers):
        for f in BlockParams.TENSOR_FIELDS:
            shapes.append((f"block{i}.{f}", blk[f]))
    shapes += [("final_gain", (d,)), ("final_bias", (d,)), ("head", (d, cfg.vocab_or_classes))]
    off = 44
    vals = {}
    for name, shp in shapes:
        n = int(np.prod(shp))
        vals[name] = np.frombuffer(blob, dtype="<f4", count=n, offset=off).reshape(shp).copy()
        off += 4 * n
    blocks = [BlockParams(*(Tensor(vals[f"block{i}.{f}"]) for f in BlockParams.TENSOR_FIELDS))
              for i in range(cfg.layers)]
    params = ModelParams(config=cfg, pos=Tensor(vals["pos"]), blocks=blocks,
                         final_gain=Tensor(vals["final_gain"]),
                         final_bias=Tensor(vals["final_bias"]), head=Tensor(vals["head"]),
                         embedding=Tensor(vals["embedding"]) if cfg.causal else None,
                         cls=Tensor(vals["cls"]) if not cfg.causal else None)
    (count,) = struct.unpack("<I", blob[off:off + 4])
    off += 4
    for _ in range(count):
        (size,) = struct.unpack("<I", blob[off:off + 4])
        off += 4
        cb = load_codebook(blob[off:off + size])
        off += size
        params.blocks[cb.layer_id].codebook = cb
    if off != len(blob):
        raise ValueError("trailing bytes in checkpoint")
    return params


# ---------------------------------------------------------------------------------------
# Model-level forward API (model.py:198-432), executed by the B200 runtime.
#
# The reference runs these as a single-process mask simulation (run_blocks) that is
# numerically the cluster forward (test_cluster.py:187-204 pins 1e-5); here every call goes
# through AstraRuntime with all devices of the plan on the current GPU, i.e. the same native
# kernels as cluster.run_inference.  Precision defaults to the fp32-class parity mode.

def _model_runtime(params, plan, mode, cls_mode="distributed", precision="parity",
                   require_codebooks=True):
    from .cluster import cached_runtime
    return cached_runtime(params, plan, mode=mode, cls_mode=cls_mode, precision=precision,
                          require_codebooks=require_codebooks)


def _check_noise(training, noise):
    if training and noise is not None and getattr(noise, "enabled", False) and noise.lam > 0.0:
        raise NotImplementedError("noise-augmented training forwards (NAVQ, vq.py:309-325) are "
                                  "training-side and out of scope for the inference runtime")


def _quantized(params, plan):
    quantized = params.blocks[0].codebook is not None
    for b in params.blocks:
        if (b.codebook is not None) != quantized:
            raise LifecycleError("codebooks must be initialized for all layers or none")
    if not quantized and plan.devices > 1:
        raise LifecycleError("multi-device forward requires initialized codebooks")
    return quantized


def _replicated(plan):
    """The mask simulation gives every owner a replica whatever plan.class_replication says
    (run_blocks uses class_owner_ids(plan, cls_mode) directly, model.py:217)."""
    from .cluster import ShardPlan
    if plan.class_replication:
        return plan
    return ShardPlan(tokens=plan.tokens, devices=plan.devices, ranges=plan.ranges,
                     class_replication=True)


def _emit_layers(rt, params, on_layer, quantized):
    """Call on_layer(i, info) with the reference's info keys (model.py:227-262) from the
    per-layer block inputs and codes the runtime recorded during the forward."""
    from .vq import QuantizedTokens, dequantize
    import torch
    for i, xin_dev in enumerate(rt.capture_inputs):
        x_in = rt.codes_by_image(xin_dev, rt.D)[0]
        info = {"x_in": x_in, "x_tensor": Tensor(x_in), "x_hat": None, "q": None}
        kv = rt.project_kv(i, torch.from_numpy(np.ascontiguousarray(x_in)).to(rt.device))
        info["k_full"], info["v_full"] = kv[:, :rt.D], kv[:, rt.D:]
        info["k_hat"] = info["v_hat"] = None
        if quantized:
            cb = params.blocks[i].codebook
            idx = rt.codes_by_image(rt.trace[i])[0].astype(np.int32)
            q = QuantizedTokens(layer_id=cb.layer_id, token_count=idx.shape[0], indices=idx,
                                bits_per_token=cb.bits_per_token)
            x_hat = dequantize(cb, q)
            kvh = rt.project_kv(i, torch.from_numpy(np.ascontiguousarray(x_hat)).to(rt.device))
            info.update(q=q, x_hat=x_hat, k_hat=kvh[:, :rt.D], v_hat=kvh[:, rt.D:])
        on_layer(i, info)


def _forward(rt, params, x0_or_ids, on_layer, quantized, ids=False):
    rt.trace = [] if (on_layer is not None and quantized) else None
    rt.capture_inputs = [] if on_layer is not None else None
    try:
        if ids:
            rt.set_ids(np.asarray(x0_or_ids, dtype=np.int64)[None, :])
        else:
            rt.stage_input(np.asarray(x0_or_ids, dtype=np.float32)[None])
        rt.forward()
        rt.check_errors()
        if on_layer is not None:
            _emit_layers(rt, params, on_layer, quantized)
    finally:
        rt.trace = None
        rt.capture_inputs = None


def run_blocks(params: ModelParams, plan, x0, *, training: bool = False, noise=None,
               cls_mode: str = "distributed", on_layer=None):
    """Push content (and class replicas, if any) through every block (model.py:198-265).
    Returns (content [T, D], replicas [R, D] or None) as Tensors."""
    cfg = params.config
    x = np.asarray(x0.data if hasattr(x0, "data") else x0)
    if x.shape != (plan.tokens, cfg.hidden):
        raise ShapeError(f"expected [{plan.tokens}, {cfg.hidden}] content, got {x.shape}")
    quantized = _quantized(params, plan)
    _check_noise(training, noise)
    class_owner_ids(plan, cls_mode)                       # validates cls_mode
    rt = _model_runtime(params, _replicated(plan), "blocks", cls_mode,
                        require_codebooks=quantized)
    _forward(rt, params, x, on_layer, quantized)
    content, reps = rt.stack_by_image()
    return Tensor(content[0]), (Tensor(reps[0]) if reps is not None else None)


def aggregate_class_tokens(replicas) -> Tensor:
    """Mean-pool replica states into one classification embedding (model.py:268-272)."""
    import torch
    from . import _native
    r = np.asarray(replicas.data if hasattr(replicas, "data") else replicas, np.float32)
    if r.ndim != 2:
        raise ShapeError("mean_rows requires a 2-D operand")
    if r.shape[0] < 1:
        raise ShapeError("no class-token replicas to aggregate")
    dev = torch.device("cuda", torch.cuda.current_device())
    rt = torch.from_numpy(np.ascontiguousarray(r)).to(dev)
    out = torch.empty(1, r.shape[1], device=dev)
    _native.call("astra_replica_mean", rt.data_ptr(), r.shape[0], 1, r.shape[1], out.data_ptr(),
                 torch.cuda.current_stream().cuda_stream)
    return Tensor(out.cpu().numpy())


def _embed_rows(table: np.ndarray, src: np.ndarray, pos: np.ndarray, pos_rows: np.ndarray):
    import torch
    from . import _native
    dev = torch.device("cuda", torch.cuda.current_device())
    t = torch.from_numpy(np.ascontiguousarray(table, np.float32)).to(dev)
    p = torch.from_numpy(np.ascontiguousarray(pos, np.float32)).to(dev)
    s = torch.from_numpy(np.ascontiguousarray(src, np.int32)).to(dev)
    pr = torch.from_numpy(np.ascontiguousarray(pos_rows, np.int32)).to(dev)
    out = torch.empty(len(src), t.shape[1], device=dev)
    _native.call("astra_embed_stack", t.data_ptr(), p.data_ptr(), None, s.data_ptr(), pr.data_ptr(),
                 len(src), t.shape[1], out.data_ptr(), torch.cuda.current_stream().cuda_stream)
    return Tensor(out.cpu().numpy())


def embed_classifier_inputs(params: ModelParams, x) -> Tensor:
    """x + pos[:T] (model.py:275-280)."""
    a = np.asarray(x.data if hasattr(x, "data") else x, np.float32)
    n = a.shape[0]
    if n > params.config.max_tokens:
        raise ShapeError(f"{n} tokens exceed max_tokens={params.config.max_tokens}")
    return _embed_rows(a, np.arange(n), params.pos.data, np.arange(n))


def embed_lm_inputs(params: ModelParams, ids, offset: int = 0) -> Tensor:
    """embedding[ids] + pos[offset:offset+T] (model.py:283-288)."""
    ids = np.asarray(ids, dtype=np.int64)
    if offset + ids.shape[0] > params.config.max_tokens:
        raise ShapeError("sequence exceeds max_tokens")
    v = params.embedding.data.shape[0]
    if ids.size and (ids.min() < 0 or ids.max() >= v):
        raise ShapeError("gather_rows: id out of range")
    return _embed_rows(params.embedding.data, ids, params.pos.data,
                       np.arange(offset, offset + ids.shape[0]))


def classify(params: ModelParams, plan, x, *, training: bool = False, noise=None,
             cls_mode: str = "distributed", on_layer=None) -> Tensor:
    """Logits [1, classes] from mean-pooled class replicas (model.py:291-302)."""
    if not params.config.class_token:
        raise ValueError("classify requires an encoder config (causal=False)")
    a = np.asarray(x.data if hasattr(x, "data") else x, np.float32)
    if a.shape[0] > params.config.max_tokens:
        raise ShapeError(f"{a.shape[0]} tokens exceed max_tokens={params.config.max_tokens}")
    if a.shape != (plan.tokens, params.config.hidden):
        raise ShapeError(f"expected [{plan.tokens}, {params.config.hidden}] content, got {a.shape}")
    quantized = _quantized(params, plan)
    _check_noise(training, noise)
    class_owner_ids(plan, cls_mode)
    rt = _model_runtime(params, _replicated(plan), "classify", cls_mode,
                        require_codebooks=quantized)
    _forward(rt, params, a, on_layer, quantized)
    return Tensor(rt.logits.cpu().numpy().copy())


def lm_logits(params: ModelParams, plan, ids, *, training: bool = False, noise=None,
              on_layer=None) -> Tensor:
    """Next-token logits [T, vocab] for a causal decoder (model.py:305-313)."""
    if not params.config.causal:
        raise ValueError("lm_logits requires a causal config")
    ids = np.asarray(ids, dtype=np.int64)
    if ids.shape[0] > params.config.max_tokens:
        raise ShapeError("sequence exceeds max_tokens")
    if ids.shape[0] != plan.tokens:
        raise ShapeError(f"expected {plan.tokens} ids, got {ids.shape[0]}")
    quantized = _quantized(params, plan)
    _check_noise(training, noise)
    rt = _model_runtime(params, plan, "lm", require_codebooks=quantized)
    _forward(rt, params, ids, on_layer, quantized, ids=True)
    out = rt.codes_by_image(rt.lm_out[rt.content_rows.long()], rt.classes)[0]
    return Tensor(out)


class DecodeState:
    """Per-layer KV cache seen by the decoding device (model.py:324-334): full precision for
    its own and generated tokens, dequantized for the rest of the prefill."""

    def __init__(self, k_layers: list, v_layers: list):
        self.k = [np.array(k, copy=True) for k in k_layers]
        self.v = [np.array(v, copy=True) for v in v_layers]

    def append(self, layer: int, k_row: np.ndarray, v_row: np.ndarray) -> None:
        self.k[layer] = np.concatenate([self.k[layer], k_row], axis=0)
        self.v[layer] = np.concatenate([self.v[layer], v_row], axis=0)


def prefill_decode_state(params: ModelParams, plan, prompt_ids):
    """Sequence-parallel prefill; the decoding device's KV view and the first greedy token
    (model.py:361-385), read back from the runtime's device-resident KV cache."""
    from .cluster import ShardPlan
    ids = np.asarray(prompt_ids, dtype=np.int64)
    plan = ShardPlan(tokens=plan.tokens, devices=plan.devices, ranges=plan.ranges,
                     class_replication=False)
    quantized = _quantized(params, plan)
    rt = _model_runtime(params, plan, "generate", require_codebooks=quantized)
    first = int(rt.generate(ids[None, :], 1)[0, 0])
    t = ids.shape[0]
    D = rt.D
    ks, vs = [], []
    for cache in rt.kv_cache:
        kv = cache[:t].float().cpu().numpy()
        ks.append(kv[:, :D].copy())
        vs.append(kv[:, D:].copy())
    return DecodeState(ks, vs), first


def generate(params: ModelParams, plan, prompt_ids, steps: int) -> list:
    """Greedy decoding: parallel prefill, then sequential decode on the device holding the last
    prompt token; ties resolve to the lowest id (model.py:388-402)."""
    if steps < 0:
        raise ValueError("steps must be non-negative")
    if steps == 0:
        return []
    ids = np.asarray(prompt_ids, dtype=np.int64)
    t0 = ids.shape[0]
    if t0 < plan.devices:
        raise ValueError("prompt must cover at least one token per device")
    if t0 + steps > params.config.max_tokens:
        raise ShapeError("prompt plus generated tokens exceed max_tokens")
    from .cluster import ShardPlan
    plan = ShardPlan(tokens=plan.tokens, devices=plan.devices, ranges=plan.ranges,
                     class_replication=False)
    quantized = _quantized(params, plan)
    rt = _model_runtime(params, plan, "generate", require_codebooks=quantized)
    return [int(v) for v in rt.generate(ids[None, :], steps)[0]]


def exact_codebooks_from_reference(params: ModelParams, plan1, x_or_ids) -> list:
    """Codebooks whose centroids are exactly this forward's own layer inputs, so quantization
    reproduces every token bit for bit (K = T) (model.py:405-432)."""
    if plan1.devices != 1:
        raise ValueError("reference capture requires a single-device plan")
    cfg = params.config
    stripped = ModelParams(
        config=cfg, pos=params.pos,
        blocks=[BlockParams(*(getattr(b, f) for f in BlockParams.TENSOR_FIELDS))
                for b in params.blocks],
        final_gain=params.final_gain, final_bias=params.final_bias,
        head=params.head, embedding=params.embedding, cls=params.cls)
    captured = []
    cap = lambda _i, info: captured.append(info["x_in"].copy())  # noqa: E731
    if cfg.causal:
        lm_logits(stripped, plan1, x_or_ids, on_layer=cap)
    else:
        classify(stripped, plan1, x_or_ids, on_layer=cap)
    gd = cfg.hidden // cfg.groups
    return [Codebook(layer_id=layer, groups=cfg.groups,
                     centroids=[np.ascontiguousarray(xin[:, g * gd:(g + 1) * gd])
                                for g in range(cfg.groups)])
            for layer, xin in enumerate(captured)]
