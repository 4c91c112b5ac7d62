"""Shared test helpers (configs from golden JSON, store digests)."""

from __future__ import annotations

import hashlib

from paper_2605_22014_b200.specs import ModelSpec, ParallelConfig


def cfg_from_json(d: dict) -> ParallelConfig:
    return ParallelConfig(d["gen"], d["tp"], d["pp"], d["dp"], list(d["ranks"]), d.get("layer_stage"))


def spec_from_text(text: str) -> ModelSpec:
    return ModelSpec.from_text(text)


def sha(s) -> str:
    if isinstance(s, str):
        s = s.encode()
    return hashlib.sha256(s).hexdigest()


def engine_store_digest(engine, which: int, model: ModelSpec, owners) -> str:
    """sha256 over 'ti:rank:' + bytes in (ti, rank) order -- the golden digest format."""
    h = hashlib.sha256()
    for ti, rank in owners:
        h.update(f"{ti}:{rank}:".encode())
        _, n = engine.ptr(which, rank, ti)
        off = 0
        while off < n:
            step = min(n - off, 256 << 20)
            h.update(engine.read(which, rank, ti, off, step).tobytes())
            off += step
    return h.hexdigest()


def oracle_owners(store) -> list:
    return sorted(store.entries.keys())
