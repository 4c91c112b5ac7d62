"""One process per GPU: torch.distributed plumbing for the reshard engine.

torch.distributed is only the control plane here (rendezvous, all-gather of
64-byte CUDA IPC handles, barriers).  Every byte of model state moves through
the engine's kernels over peer mappings (NVLink), never through a collective.

    eng = R.Engine([local_gpu], world_slots=world, first_local_slot=rank, ...)
    eng.layout(RS_SRC, model, c_old, slot_of_old_rank)   # same on every rank
    eng.layout(RS_DST, model, c_new, slot_of_new_rank)
    eng.alloc(RS_SRC); eng.alloc(RS_DST); eng.comm_alloc()
    connect(eng)                                          # import every peer arena
    eng.prepare(plan); eng.run(); dist.barrier()
"""

from __future__ import annotations

from typing import Iterable, Optional

from .native import RS_COMM, RS_DST, RS_SRC


def local_slots(engine) -> list:
    return list(range(engine.first_local_slot, engine.first_local_slot + engine.num_devices))


def connect(engine, group=None, which: Iterable[int] = (RS_SRC, RS_DST, RS_COMM)) -> None:
    """Export this rank's arenas, all-gather the handles, import every peer's."""
    import torch.distributed as dist
    mine = {}
    for w in which:
        for slot in local_slots(engine):
            mine[(int(w), slot)] = engine.export_arena(w, slot)
    everyone = [None] * dist.get_world_size(group)
    dist.all_gather_object(everyone, mine, group=group)
    for table in everyone:
        for (w, slot), (handle, nbytes) in table.items():
            engine.import_arena(w, slot, handle, nbytes)


def slot_map(config, ranks_per_slot: Optional[int] = None, nslots: Optional[int] = None) -> list:
    """Placement helper: rank-list position i -> slot i // ranks_per_slot."""
    n = config.world
    if ranks_per_slot is None:
        ranks_per_slot = max(1, -(-n // (nslots or n)))
    return [i // ranks_per_slot for i in range(n)]
