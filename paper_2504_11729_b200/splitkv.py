"""Cross-GPU split-KV attention for long cloud prompts (BASELINE config 4).

The reference fuses ANY ordered partition of a row's keys exactly:
merge_partials folds per-segment (out, lse) pairs with log_add_exp in segment
order (/root/reference/proj/core/src/attention.cpp:116-156).
Here the partition is across the GPUs of one box:

* ``shard_segments`` — rank r owns the contiguous cloud slice
  [r*C/P, (r+1)*C/P); the edge (and generated) segments live on rank P-1,
  keeping the global positions so the causal rule (attention.cpp:29-33) is
  unchanged;
* every rank runs the spliced kernel (K1/K3) over its shard with fp32 output
  and lse;
* one NCCL all-gather of the packed [o | lse] buffer (torch.distributed
  plumbing), then the K5 merge kernel in rank (= segment) order on every rank
  — deterministic, identical on all ranks.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

from ._capi import check, lib


@dataclass
class Shard:
    origin: int
    pos_offset: int
    length: int


def shard_segments(segments, world: int, rank: int):
    """segments: ordered [(origin, length)] of one request starting at
    position 0. Cloud segments (origin 0) are split into `world` contiguous
    slices; non-cloud segments go to the last rank. Returns this rank's
    [Shard] (possibly empty)."""
    out = []
    pos = 0
    cloud_total = sum(l for o, l in segments if o == 0)
    cloud_seen = 0
    lo = cloud_total * rank // world
    hi = cloud_total * (rank + 1) // world
    for origin, length in segments:
        if origin == 0:
            a, b = max(lo, cloud_seen), min(hi, cloud_seen + length)
            if b > a:
                out.append(Shard(0, pos + (a - cloud_seen), b - a))
            cloud_seen += length
        elif rank == world - 1:
            out.append(Shard(origin, pos, length))
        pos += length
    return out


class SplitKVCombine:
    """All-gather of every rank's fp32 (o, lse) + the K5 LSE merge.

    ``gather(tensor_out, tensor_in)`` defaults to
    torch.distributed.all_gather_into_tensor on the default (NCCL) group;
    ``merge(packed, world, rows, d) -> (o, lse)`` defaults to the K5 kernel
    (ep_merge_partials_packed_dev). Both are injectable so the host logic can
    be exercised on CPU (gloo) in tests."""

    def __init__(self, world: int, rows: int, d: int, handle=None, gather=None, merge=None,
                 device=None):
        import torch
        self.world, self.rows, self.d = world, rows, d
        self.handle = handle
        self._gather = gather
        self._merge = merge
        self.device = device
        n = rows * (d + 1)
        self.send = torch.empty(n, dtype=torch.float32, device=device)
        self.recv = torch.empty(world * n, dtype=torch.float32, device=device)

    def __call__(self, o_part, lse_part, out=None, out_lse=None, stream=None):
        """o_part [rows*d] / [.., d] fp32 and lse_part [rows] (natural log) of
        this rank's keys -> merged (o [rows][d], lse [rows])."""
        import torch
        rd = self.rows * self.d
        self.send[:rd].copy_(o_part.reshape(-1))
        self.send[rd:].copy_(lse_part.reshape(-1))
        if self._gather is None:
            import torch.distributed as dist
            dist.all_gather_into_tensor(self.recv, self.send)
        else:
            self._gather(self.recv, self.send)
        if self._merge is not None:
            return self._merge(self.recv, self.world, self.rows, self.d)
        if out is None:
            out = torch.empty((self.rows, self.d), dtype=torch.float32, device=self.recv.device)
        if out_lse is None:
            out_lse = torch.empty((self.rows,), dtype=torch.float32, device=self.recv.device)
        odt = {torch.float32: 0, torch.bfloat16: 1}[out.dtype]
        s = torch.cuda.current_stream().cuda_stream if stream is None else getattr(
            stream, "cuda_stream", stream)
        check(lib().ep_merge_partials_packed_dev(self.handle.ptr, self.world,
                                                 self.recv.data_ptr(), self.rows, self.d, odt,
                                                 out.data_ptr(), out_lse.data_ptr(), s),
              "ep_merge_partials_packed_dev")
        return out, out_lse
