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


class PeerSplitKVCombine:
    """The combine as ONE kernel over NVLink peer memory
    (ep_splitkv_combine_dev): every rank pushes its fp32 (o, lse) rows into
    the peers' receive buffers and merges what it received in rank order — no
    NCCL on the data path. The group's buffers are exchanged once:

    * across processes (one per GPU): ``PeerSplitKVCombine(world, rank, rows,
      d, handle)`` exchanges CUDA IPC handles with
      torch.distributed.all_gather_object (``exchange`` is injectable);
    * inside one process (tests: P emulated ranks on one GPU, or a thread per
      GPU): ``PeerSplitKVCombine.local_group(world, rows, d, handles)``.
    """

    def __init__(self, world: int, rank: int, rows: int, d: int, handle, exchange=None,
                 _connect=True):
        self.world, self.rank, self.rows, self.d = world, rank, rows, d
        self.handle = handle
        self._lib = lib()
        g = C.c_void_p()
        check(self._lib.ep_peer_group_create(handle.ptr, world, rank, rows, d, C.byref(g)),
              "ep_peer_group_create")
        self._g = g
        if _connect and world > 1:
            buf = (C.c_ubyte * 64)()
            check(self._lib.ep_peer_group_export(g, buf), "ep_peer_group_export")
            mine = bytes(buf)
            if exchange is None:
                import torch.distributed as dist
                handles = [None] * world
                dist.all_gather_object(handles, mine)
            else:
                handles = exchange(mine)
            assert len(handles) == world and all(len(x) == 64 for x in handles)
            blob = b"".join(handles)
            check(self._lib.ep_peer_group_connect_ipc(g, blob), "ep_peer_group_connect_ipc")
            if exchange is None:
                import torch.distributed as dist
                dist.barrier()

    @classmethod
    def local_group(cls, world: int, rows: int, d: int, handles):
        """world groups in this process (handles[r] = rank r's Handle; may share a device)."""
        groups = [cls(world, r, rows, d, handles[r], _connect=False) for r in range(world)]
        bases = (C.c_void_p * world)()
        for r, g in enumerate(groups):
            b = C.c_void_p()
            check(g._lib.ep_peer_group_base(g._g, C.byref(b)), "ep_peer_group_base")
            bases[r] = b
        if world > 1:
            for g in groups:
                check(g._lib.ep_peer_group_connect_ptrs(g._g, bases), "ep_peer_group_connect_ptrs")
        return groups

    def __call__(self, o_part, lse_part, out=None, out_lse=None, stream=None):
        """o_part [rows][d] fp32, lse_part [rows] fp32 (natural log) of this rank's
        keys -> merged (out [rows][d] fp32/bf16, out_lse [rows])."""
        import torch
        assert o_part.dtype == torch.float32 and lse_part.dtype == torch.float32
        assert o_part.is_contiguous() and lse_part.is_contiguous()
        dev = o_part.device
        if out is None:
            out = torch.empty((self.rows, self.d), dtype=torch.float32, device=dev)
        if out_lse is None:
            out_lse = torch.empty((self.rows,), dtype=torch.float32, device=dev)
        odt = {torch.float32: 0, torch.bfloat16: 1}[out.dtype]
        s = torch.cuda.current_stream(dev).cuda_stream if stream is None else getattr(
            stream, "cuda_stream", stream)
        check(self._lib.ep_splitkv_combine_dev(self.handle.ptr, self._g, self.rows,
                                               o_part.data_ptr(), lse_part.data_ptr(), odt,
                                               out.data_ptr(), out_lse.data_ptr(), s),
              "ep_splitkv_combine_dev")
        return out, out_lse

    def attend(self, attn, q, out=None, out_lse=None, stream=None):
        """Split-KV attention with the combine fused into the decode kernel
        (ep_spliced_attention_splitkv): ``attn`` is this rank's
        SplicedAttention over its KV shard; one launch computes the shard's
        partials, exchanges them over NVLink and merges them in rank order.
        Returns (out [B][n_q][Hq][d], out_lse [B][n_q][Hq]) — identical on every
        rank. A group serves either this or __call__ (the separate combine
        kernel), not both."""
        import torch
        from .splice import _stream, dtype_code
        if out is None:
            out = torch.empty(q.shape, dtype=q.dtype, device=q.device)
        if out_lse is None:
            out_lse = torch.empty(tuple(q.shape[:3]), dtype=torch.float32, device=q.device)
        pd = attn.pool.desc()
        check(self._lib.ep_spliced_attention_splitkv(self.handle.ptr, attn.plan, C.byref(pd), dtype_code(q.dtype),
                                                     q.data_ptr(), self._g, dtype_code(out.dtype), out.data_ptr(),
                                                     out_lse.data_ptr() if out_lse is not False else None,
                                                     _stream(stream)),
              "ep_spliced_attention_splitkv")
        return out, out_lse

    def close(self):
        if self._g is not None and self._g.value:
            self._lib.ep_peer_group_destroy(self._g)
        self._g = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


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
