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


class ShardedExtractor:
    """Host protocol of a sharded multi-GPU extraction (ssbh_shard_*, one process per GPU).

    Rank r samples only its slice of rounds; the sampled payload goes straight into the
    owning rank's receive buffer through NVLink peer memory (IPC mappings exchanged once
    here); each rank then builds and hashes its own blocks. torch.distributed carries only
    the handles (once), a W x W count matrix and a barrier per run."""

    def __init__(self, n, s, k, samp, hsh, per_block=False, group=None):
        import torch.distributed as dist

        import paper_2308_02856_b200 as P

        self.dist, self.group = dist, group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.shard = P.Shard(n, s, k, samp, hsh, self.rank, self.world, per_block=per_block)
        handles = [None] * self.world
        dist.all_gather_object(handles, self.shard.ipc_handle(), group=group)
        self.shard.open_peers(handles)
        self.n, self.s, self.k = n, s, k

    @property
    def slice(self):
        return self.shard.slice_first, self.shard.slice_rounds

    @property
    def blocks(self):
        return self.shard.block_first, self.shard.block_count

    def run(self, d_slice_ptr: int, d_key_ptr: int, d_len_ptr: int = 0, stream: int = 0,
            coll_device: str = "cpu"):
        import torch

        counts = self.shard.sample(d_slice_ptr, stream)
        mine = torch.from_numpy(counts.view(np.int64).copy()).to(coll_device)
        rows = [torch.empty_like(mine) for _ in range(self.world)]
        self.dist.all_gather(rows, mine, group=self.group)
        matrix = np.stack([r.cpu().numpy().view(np.uint64) for r in rows])
        self.shard.exchange(matrix, stream)
        self.dist.barrier(group=self.group)  # every rank's peer stores have landed
        self.shard.finish(d_key_ptr, d_len_ptr, stream)
        return matrix

    def check(self):
        return self.shard.check()

    def close(self):
        self.dist.barrier(group=self.group)  # peers are done with our receive buffer
        self.shard.close()


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
