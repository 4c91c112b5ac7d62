"""Canonical model specs and parallel configs for the reshard path.

The reference models training state as a ``ModelSpec`` of ``TensorSpec``
(``proj/include/reshard/model_spec.hpp:26-87``) and a layout as a
``ParallelConfig`` (``proj/include/reshard/parallel_config.hpp:27-70``).  This
module builds those descriptions for the BASELINE.json architectures and
serialises them into the one text format every component here reads: the
product planner (``csrc/model.cpp``), the C oracle (``oracle/oracle.c``) and the
reference harness (``oracle/ref_harness.cpp``).

Spec text format (one record per line, ``#`` comments)::

    model <name> layers <L> bpe <default bytes per element>
    tensor <id> <layer> <d0,d1,...> <tp axis | -> <param|m1|m2> <bytes per element>

Tensor order is semantic: the synthetic fill pattern depends on the tensor's
index in the spec (``proj/src/shard_store.cpp:51-56``), so the builders below
are the single source of tensor order.

Per-tensor element size is an extension over the reference (one
``bytes_per_element`` per model, ``model_spec.hpp:45``).  A spec whose tensors
all share one size is exactly a reference spec; ``group_spec`` splits a mixed
spec into such single-size groups for reference parity.
"""

from __future__ import annotations

import dataclasses
import random
from typing import Iterable, List, Optional, Sequence

ROLES = ("param", "m1", "m2")


@dataclasses.dataclass
class TensorSpec:
    tensor_id: str
    layer: int
    shape: List[int]
    tp_shard_axis: Optional[int]
    role: str = "param"
    bpe: int = 4
    dp_axis: Optional[int] = None  # extension: distributed-optimizer DP split axis

    def element_count(self) -> int:
        n = 1
        for d in self.shape:
            n *= d
        return n

    def nbytes(self) -> int:
        return self.element_count() * self.bpe


@dataclasses.dataclass
class ModelSpec:
    name: str
    num_layers: int
    tensors: List[TensorSpec]
    bytes_per_element: int = 4

    def to_text(self) -> str:
        out = [f"model {self.name} layers {self.num_layers} bpe {self.bytes_per_element}"]
        for t in self.tensors:
            axis = "-" if t.tp_shard_axis is None else str(t.tp_shard_axis)
            shape = ",".join(str(d) for d in t.shape)
            dp = "" if t.dp_axis is None else f" dp={t.dp_axis}"
            out.append(f"tensor {t.tensor_id} {t.layer} {shape} {axis} {t.role} {t.bpe}{dp}")
        return "\n".join(out) + "\n"

    @staticmethod
    def from_text(text: str) -> "ModelSpec":
        spec = None
        tensors: List[TensorSpec] = []
        for raw in text.splitlines():
            line = raw.split("#", 1)[0].strip()
            if not line:
                continue
            tok = line.split()
            if tok[0] == "model":
                spec = ModelSpec(tok[1], int(tok[3]), tensors, int(tok[5]))
            elif tok[0] == "tensor":
                axis = None if tok[4] == "-" else int(tok[4])
                dp = None
                for opt in tok[7:]:
                    if opt.startswith("dp="):
                        dp = int(opt[3:])
                tensors.append(TensorSpec(tok[1], int(tok[2]),
                                          [int(x) for x in tok[3].split(",")],
                                          axis, tok[5], int(tok[6]), dp))
            else:
                raise ValueError(f"spec parse: unknown record {tok[0]!r}")
        if spec is None:
            raise ValueError("spec parse: missing model record")
        return spec

    def total_bytes(self) -> int:
        return sum(t.nbytes() for t in self.tensors)

    def uniform_bpe(self) -> Optional[int]:
        sizes = {t.bpe for t in self.tensors}
        return sizes.pop() if len(sizes) == 1 else None


@dataclasses.dataclass
class ParallelConfig:
    """(tp, pp, dp) over an ordered rank list; ``parallel_config.hpp:21-23``."""

    gen: int
    tp: int
    pp: int
    dp: int
    ranks: List[int]
    layer_stage: Optional[List[int]] = None  # None: default ceil split
    # extension: DP-shard the tensors that declare a dp_axis (ZeRO-1):
    # 0/False off, 1/True per-tensor dim chunks, 2 Megatron flat buckets
    dist_opt: int = 0
    bucket_elems: int = 0  # flat buckets: bucket size in elements (0: max(40M, 1M x dp))

    @property
    def world(self) -> int:
        return len(self.ranks)

    def stages(self, num_layers: int) -> List[int]:
        if self.layer_stage is not None:
            return list(self.layer_stage)
        return default_layer_assignment(num_layers, self.pp)

    def describe(self) -> str:
        return f"TP{self.tp}PP{self.pp}DP{self.dp}"


def default_layer_assignment(num_layers: int, pp: int) -> List[int]:
    """Contiguous ceil split, earlier stages heavier (``parallel_config.cpp:19-29``)."""
    base, extra = divmod(num_layers, pp)
    out: List[int] = []
    for s in range(pp):
        out += [s] * (base + (1 if s < extra else 0))
    return out[:num_layers]


def iota_config(gen: int, tp: int, pp: int, dp: int, first: int = 0,
                layer_stage: Optional[List[int]] = None) -> ParallelConfig:
    return ParallelConfig(gen, tp, pp, dp, list(range(first, first + tp * pp * dp)),
                          layer_stage)


def group_spec(spec: ModelSpec, bpe: int) -> ModelSpec:
    """The single-element-size sub-spec a reference ``ModelSpec`` can express."""
    ts = [dataclasses.replace(t) for t in spec.tensors if t.bpe == bpe]
    return ModelSpec(f"{spec.name}[{bpe}B]", spec.num_layers, ts, bpe)


# ---------------------------------------------------------------------------
# Architectures.  Megatron-style layouts:
#   column-parallel [out, in] axis 0; row-parallel [out, in] axis 1;
#   vocab-parallel embedding/head [V, h] axis 0;
#   fused QKV group-interleaved [ng, q_per_g + 2, hd, h] axis 0;
#   SwiGLU fc1 stored per rank as [gate_r; up_r] -> [2, ffn, h] axis 1.
# ---------------------------------------------------------------------------

def dp_axis_for(shape: Sequence[int]) -> int:
    """Distributed-optimizer split axis: the first axis of extent >= 64 (chunks
    stay large and balanced: embed/head rows, QKV head_dim, fc1 ffn), else 0."""
    for i, d in enumerate(shape):
        if d >= 64:
            return i
    return 0


def _emit(tensors: List[TensorSpec], layer: int, name: str, shape: Sequence[int],
          axis: Optional[int], state: Sequence[tuple], zero: bool = False) -> None:
    for suffix, role, bpe in state:
        # ZeRO-1: fp32 optimizer state (master, m, v) is DP-sharded, bf16
        # weights stay DP-replicated
        dp = dp_axis_for(shape) if zero and bpe == 4 and suffix != "param" else None
        tensors.append(TensorSpec(f"L{layer}.{name}.{suffix}", layer, list(shape), axis,
                                  role, bpe, dp))


def gpt2_124m(num_layers: int = 12) -> ModelSpec:
    """GPT-2 small, fp32 params + Adam m/v (BASELINE config 1)."""
    h, heads, ffn, vocab, npos = 768, 12, 3072, 50257, 1024
    hd = h // heads
    state = (("param", "param", 4), ("m1", "m1", 4), ("m2", "m2", 4))
    ts: List[TensorSpec] = []
    for l in range(num_layers):
        if l == 0:
            _emit(ts, l, "wte", (vocab, h), 0, state)
            _emit(ts, l, "wpe", (npos, h), None, state)
        _emit(ts, l, "ln1.w", (h,), None, state)
        _emit(ts, l, "ln1.b", (h,), None, state)
        _emit(ts, l, "attn.qkv.w", (heads, 3, hd, h), 0, state)
        _emit(ts, l, "attn.qkv.b", (heads, 3, hd), 0, state)
        _emit(ts, l, "attn.proj.w", (h, h), 1, state)
        _emit(ts, l, "attn.proj.b", (h,), None, state)
        _emit(ts, l, "ln2.w", (h,), None, state)
        _emit(ts, l, "ln2.b", (h,), None, state)
        _emit(ts, l, "mlp.fc1.w", (ffn, h), 0, state)
        _emit(ts, l, "mlp.fc1.b", (ffn,), 0, state)
        _emit(ts, l, "mlp.fc2.w", (h, ffn), 1, state)
        _emit(ts, l, "mlp.fc2.b", (h,), None, state)
        if l == num_layers - 1:
            _emit(ts, l, "lnf.w", (h,), None, state)
            _emit(ts, l, "lnf.b", (h,), None, state)
            # tied head, modelled as a separate last-stage tensor
            _emit(ts, l, "head", (vocab, h), 0, state)
    return ModelSpec(f"gpt2-124m-L{num_layers}", num_layers, ts, 4)


LLAMA = {
    # name: (hidden, layers, q heads, kv heads, head dim, ffn, vocab)
    "llama2-7b": (4096, 32, 32, 32, 128, 11008, 32000),
    "llama3-8b": (4096, 32, 32, 8, 128, 14336, 128256),
    "llama2-13b": (5120, 40, 40, 40, 128, 13824, 32000),
    # test scale: same tensor structure (GQA fused QKV, SwiGLU fc1), tiny dims
    "llama-mini": (256, 4, 16, 8, 16, 688, 1000),
    # same, with ffn / vocab multiples of 64: every TP split of every tensor is
    # a 16 B-aligned run, so the default DIRECT kernel is the TMA bulk copy
    "llama-mini-a16": (256, 4, 16, 8, 16, 704, 1024),
}

# bf16 model weights + fp32 master weights + fp32 Adam m / v
MIXED_STATE = (("param", "param", 2), ("master", "param", 4), ("m1", "m1", 4),
               ("m2", "m2", 4))


def llama(arch: str, num_layers: Optional[int] = None,
          state: Sequence[tuple] = MIXED_STATE, zero: bool = False) -> ModelSpec:
    """Llama family spec.  zero=True annotates the fp32 optimizer state for the
    distributed optimizer (it is DP-sharded under a config with dist_opt)."""
    h, layers, nq, nkv, hd, ffn, vocab = LLAMA[arch]
    L = layers if num_layers is None else num_layers
    ts: List[TensorSpec] = []
    qpg = nq // nkv
    for l in range(L):
        if l == 0:
            _emit(ts, l, "embed", (vocab, h), 0, state, zero)
        _emit(ts, l, "input_norm", (h,), None, state, zero)
        _emit(ts, l, "attn.qkv", (nkv, qpg + 2, hd, h), 0, state, zero)
        _emit(ts, l, "attn.o", (h, nq * hd), 1, state, zero)
        _emit(ts, l, "post_norm", (h,), None, state, zero)
        _emit(ts, l, "mlp.fc1", (2, ffn, h), 1, state, zero)
        _emit(ts, l, "mlp.fc2", (h, ffn), 1, state, zero)
        if l == L - 1:
            _emit(ts, l, "final_norm", (h,), None, state, zero)
            _emit(ts, l, "lm_head", (vocab, h), 0, state, zero)
    default = 4 if any(s[2] == 4 for s in state) else state[0][2]
    suffix = "" if num_layers is None else f"-L{L}"
    return ModelSpec(f"{arch}{suffix}{'-zero' if zero else ''}", L, ts, default)


# ---------------------------------------------------------------------------
# BASELINE.json configurations (iota rank lists)
# ---------------------------------------------------------------------------

def baseline_case(name: str):
    """Returns (spec, c_old, c_new) for a named BASELINE configuration."""
    if name == "c1":  # GPT-2 TP2PP2DP2 -> TP4PP2DP1, 8 ranks
        return gpt2_124m(), iota_config(1, 2, 2, 2), iota_config(2, 4, 2, 1)
    if name == "c2":  # Llama-2-7B TP4PP2 (8) -> TP2PP2 (4)
        return llama("llama2-7b"), iota_config(1, 4, 2, 1), iota_config(2, 2, 2, 1)
    if name == "c3":  # Llama-3-8B TP8 -> TP4DP2 (reference replicated-DP semantics)
        return llama("llama3-8b"), iota_config(1, 8, 1, 1), iota_config(2, 4, 1, 2)
    if name == "c3z":  # BASELINE config 3 proper: TP8 -> TP4DP2 with the distributed
        # optimizer re-partitioning fp32 master/m/v across the 2 DP ranks (extension)
        c_new = dataclasses.replace(iota_config(2, 4, 1, 2), dist_opt=True)
        return llama("llama3-8b", zero=True), iota_config(1, 8, 1, 1), c_new
    if name == "c3zb":  # the same with Megatron's flat-bucket distributed optimizer layout:
        # DP ranks hold contiguous ranges of 40M-element buckets (extension)
        c_new = dataclasses.replace(iota_config(2, 4, 1, 2), dist_opt=2)
        return llama("llama3-8b", zero=True), iota_config(1, 8, 1, 1), c_new
    if name == "c4":  # Llama-2-13B TP2PP4 -> TP4PP2 with uneven 21/19 split
        spec = llama("llama2-13b")
        return spec, iota_config(1, 2, 4, 1), iota_config(2, 4, 2, 1, layer_stage=[0] * 21 + [1] * 19)
    if name == "c5":  # Llama-2-7B TP2PP2 (4) -> TP4PP2 (8)
        return llama("llama2-7b"), iota_config(1, 2, 2, 1), iota_config(2, 4, 2, 1)
    if name == "c5b":  # Llama-2-7B TP2PP2 (4) -> TP2PP2DP2 (8)
        return llama("llama2-7b"), iota_config(1, 2, 2, 1), iota_config(2, 2, 2, 2)
    raise KeyError(name)


def sliced_case(name: str, num_layers: int):
    """The same resize on an ``num_layers``-deep slice of the architecture."""
    spec, c_old, c_new = baseline_case(name)
    if name == "c1":
        spec = gpt2_124m(num_layers)
    else:
        arch = {"c2": "llama2-7b", "c3": "llama3-8b", "c3z": "llama3-8b", "c3zb": "llama3-8b", "c4": "llama2-13b",
                "c5": "llama2-7b", "c5b": "llama2-7b"}[name]
        spec = llama(arch, num_layers, zero=name in ("c3z", "c3zb"))
    c_old = dataclasses.replace(c_old, layer_stage=None)
    c_new = dataclasses.replace(c_new, layer_stage=None)
    if name == "c4" and num_layers >= 3:
        # keep C4's point: an uneven PP2 stage migration (21/19 of 40 layers at
        # full size -> ceil(21 L / 40), never an even split, on an L-layer slice)
        first = -(-21 * num_layers // 40)
        if 2 * first == num_layers:
            first += 1
        c_new = dataclasses.replace(c_new, layer_stage=[0] * first + [1] * (num_layers - first))
    return spec, c_old, c_new


# ---------------------------------------------------------------------------
# Random toy pairs (<= 8 layers, dims <= 64, world <= 16)
# ---------------------------------------------------------------------------

def _factor3(rng: random.Random, world: int, max_pp: int):
    choices = []
    for tp in range(1, world + 1):
        for pp in range(1, min(max_pp, world) + 1):
            if world % (tp * pp) == 0:
                choices.append((tp, pp, world // (tp * pp)))
    return rng.choice(choices)


def _rand_stages(rng: random.Random, L: int, pp: int) -> Optional[List[int]]:
    if rng.random() < 0.5:
        return None
    cuts = sorted(rng.sample(range(1, L), pp - 1)) if pp > 1 else []
    out, s = [], 0
    for l in range(L):
        while s < len(cuts) and l >= cuts[s]:
            s += 1
        out.append(s)
    return out


def random_case(seed: int):
    """One random (spec, c_old, c_new) triple spanning in-place / scale-out / scale-in."""
    rng = random.Random(seed)
    L = rng.randint(1, 8)
    kind = rng.choice(("inplace", "scale_out", "scale_in"))
    w_old = rng.randint(1, 16)
    if kind == "inplace":
        w_new = w_old
    elif kind == "scale_out":
        w_new = rng.randint(w_old, 16)
    else:
        w_new = rng.randint(1, w_old)
    tp0, pp0, dp0 = _factor3(rng, w_old, L)
    tp1, pp1, dp1 = _factor3(rng, w_new, L)
    pool = rng.sample(range(24), max(w_old, w_new))
    if kind == "scale_in":
        old_ranks = pool[:w_old]
        new_ranks = rng.sample(old_ranks, w_new)
    else:
        new_ranks = pool[:w_new]
        old_ranks = rng.sample(new_ranks, w_old)
    c_old = ParallelConfig(1, tp0, pp0, dp0, old_ranks, _rand_stages(rng, L, pp0))
    c_new = ParallelConfig(2, tp1, pp1, dp1, new_ranks, _rand_stages(rng, L, pp1))
    bpe = rng.choice((1, 2, 4))
    min_axis = max(tp0, tp1)
    ts: List[TensorSpec] = []
    for l in range(L):
        for k in range(rng.randint(1, 3)):
            nd = rng.randint(1, 3)
            axis = rng.choice([None] + list(range(nd)))
            shape = []
            for d in range(nd):
                lo = min_axis if d == axis else 1
                shape.append(rng.randint(lo, max(lo, 64 if nd == 1 else 24)))
            ts.append(TensorSpec(f"t{l}_{k}", l, shape, axis, rng.choice(ROLES), bpe))
    spec = ModelSpec(f"toy{seed}", L, ts, bpe)
    return spec, c_old, c_new


def iter_random_cases(n: int, base_seed: int = 20260517) -> Iterable[tuple]:
    for i in range(n):
        yield (base_seed + i,) + random_case(base_seed + i)


def random_zero_case(seed: int):
    """A random pair with distributed-optimizer sharding (extension): some
    tensors get a dp axis, and either config may enable dist_opt."""
    spec, c_old, c_new = random_case(seed)
    rng = random.Random(seed ^ 0x5EED)
    for t in spec.tensors:
        if rng.random() < 0.6:
            t.dp_axis = rng.randrange(len(t.shape))
    c_old = dataclasses.replace(c_old, dist_opt=rng.random() < 0.6)
    c_new = dataclasses.replace(c_new, dist_opt=rng.random() < 0.6)
    return spec, c_old, c_new


def iter_random_zero_cases(n: int, base_seed: int = 31337) -> Iterable[tuple]:
    for i in range(n):
        yield (base_seed + i,) + random_zero_case(base_seed + i)


def random_flat_case(seed: int):
    """A random pair where either config may use the Megatron flat-bucket
    distributed optimizer (dist_opt 2) with a small random bucket size, so
    buckets close mid-stage and DP ranges cut tensors mid-row (extension)."""
    spec, c_old, c_new = random_zero_case(seed)
    rng = random.Random(seed ^ 0xF1A7)
    modes = (0, 1, 2, 2)
    c_old = dataclasses.replace(c_old, dist_opt=rng.choice(modes), bucket_elems=rng.choice((0, 64, 200, 777, 5000)))
    c_new = dataclasses.replace(c_new, dist_opt=rng.choice(modes[1:]) if c_old.dist_opt != 2 else rng.choice(modes),
                                bucket_elems=rng.choice((0, 64, 200, 777, 5000)))
    return spec, c_old, c_new


def iter_random_flat_cases(n: int, base_seed: int = 4242) -> Iterable[tuple]:
    for i in range(n):
        yield (base_seed + i,) + random_flat_case(base_seed + i)
