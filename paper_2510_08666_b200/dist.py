"""Host-side plumbing for the vocab-sharded step (torch.distributed).

* `shard_range(V, rank, world)`: contiguous vocab rows of W_vocab / E per rank.
* `broadcast_unique_id(device)`: rank 0 draws the 128-byte NCCL unique id
  through the C ABI (dinfer_get_unique_id) and broadcasts it over the default
  process group (nccl or gloo) so every rank can create its communicator.
"""
from __future__ import annotations

from .synth import shard_range  # noqa: F401  (one definition of the shard split)


def broadcast_unique_id(device="cpu", id_bytes: bytes | None = None) -> bytes:
    import torch
    import torch.distributed as dist
    buf = torch.zeros(128, dtype=torch.uint8, device=device)
    if dist.get_rank() == 0:
        if id_bytes is None:
            from .dinfer import get_unique_id
            id_bytes = get_unique_id()
        buf.copy_(torch.frombuffer(bytearray(id_bytes), dtype=torch.uint8).to(device))
    dist.broadcast(buf, 0)
    return bytes(buf.cpu().numpy().tobytes())
