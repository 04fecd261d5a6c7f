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

from .errors import ShapeError
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
