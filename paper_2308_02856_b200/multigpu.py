"""Multi-GPU host logic: sub-block ownership and gathering of the concatenated key.

Sub-blocks are independent, so each rank owns a contiguous
block range and hashes it with no data-path collective; the only exchange is gathering
the owned key slices in block order (what BitString::append does,
proj/src/bitstring.cpp:42-47). One process per GPU, torch.distributed for the plumbing
(NCCL on GPUs, gloo in the CPU tests).
"""
from __future__ import annotations

import numpy as np


def owned_range(rank: int, world: int, n_subblocks: int) -> tuple[int, int]:
    """Contiguous, balanced block range [first, first + count) of `rank`."""
    if not (0 <= rank < world):
        raise ValueError("rank out of range")
    first = rank * n_subblocks // world
    return first, (rank + 1) * n_subblocks // world - first


def concat_bits(parts: list[np.ndarray], bit_lengths: list[int]) -> np.ndarray:
    """Concatenate LSB-first uint64 word arrays holding bit_lengths[i] bits each."""
    total = int(sum(bit_lengths))
    out = np.zeros(max((total + 63) // 64, 1), dtype=np.uint64)
    pos = 0
    for words, nb in zip(parts, bit_lengths):
        if nb == 0:
            continue
        bits = np.unpackbits(np.ascontiguousarray(words, dtype=np.uint64).view(np.uint8),
                             bitorder="little")[:nb]
        dst = np.unpackbits(out.view(np.uint8), bitorder="little")
        dst[pos:pos + nb] = bits
        out = np.packbits(dst, bitorder="little").view(np.uint64)
        pos += nb
    return out[: (total + 63) // 64]


def gather_key(local_words, n_subblocks: int, out_bits: int, group=None):
    """All-gather every rank's owned key slice (torch int64 tensor of uint64 words) and return
    the full concatenated key as uint64 numpy words on every rank."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    counts = [owned_range(r, world, n_subblocks)[1] for r in range(world)]
    lens = [(c * out_bits + 63) // 64 for c in counts]
    width = max(lens) if lens else 0
    buf = torch.zeros(width, dtype=torch.int64, device=local_words.device)
    buf[: local_words.numel()] = local_words.view(torch.int64)
    bufs = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(bufs, buf, group=group)
    parts = [b[:ln].cpu().numpy().view(np.uint64) for b, ln in zip(bufs, lens)]
    if out_bits % 64 == 0:
        return np.concatenate(parts) if parts else np.zeros(0, dtype=np.uint64)
    return concat_bits(parts, [c * out_bits for c in counts])
