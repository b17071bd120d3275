"""GPU parity of the cross-GPU split-KV path (config 4).

* On one GPU: P "ranks" are emulated as P shard plans over separate pools;
  their fp32 (o, lse) partials are packed exactly as the NCCL all-gather packs
  them and merged by the K5 kernel — compared with the unsharded spliced
  attention and with the fp64 oracle.
* The peer-memory combine kernel with P ranks emulated in one process (own
  stream each) against the K5 merge.
* With >= 2 GPUs: tools/splitkv_bench.py --check under torchrun (peer-memory
  combine over NVLink and NCCL all-gather + K5, each checked against an
  unsharded single-GPU run)."""
import os
import subprocess
import sys

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("world", [2, 4, 8])
def test_emulated_ranks_merge(cuda_handle, world):
    import torch
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import splitkv_bench as SB
    from paper_2504_11729_b200.splitkv import SplitKVCombine
    batch, cloud, edge = 3, 8192, 200
    rows, D = batch * SB.HQ, SB.D
    parts = []
    for r in range(world):
        _, _, attn, q, _ = SB.build_local(batch, world, r, cuda_handle, cloud=cloud, edge=edge)
        o, l = attn(q, o_dtype=torch.float32)
        parts.append(torch.cat([o.reshape(-1), l.reshape(-1)]))
    packed = torch.cat(parts)

    def gather(out, inp):  # the all-gather result, already assembled
        out.copy_(packed)

    comb = SplitKVCombine(world, rows, D, handle=cuda_handle, gather=gather, device="cuda")
    mo, ml = comb(parts[0][:rows * D], parts[0][rows * D:])
    _, _, attn1, q1, _ = SB.build_local(batch, 1, 0, cuda_handle, cloud=cloud, edge=edge)
    o1, l1 = attn1(q1, o_dtype=torch.float32)
    torch.cuda.synchronize()
    err = (mo - o1.reshape(rows, D)).abs().max().item()
    lerr = (ml - l1.reshape(rows)).abs().max().item()
    print(f"world {world}: merged vs unsharded max abs err {err:.2e}, lse {lerr:.2e}")
    assert err < 1e-4 and lerr < 1e-4
    # and against the fp64 oracle's merge of the same rank partials (K5 == merge_partials)
    pk = packed.cpu().numpy().astype(np.float64).reshape(world, rows * (D + 1))
    want_o, want_l = O.merge_partials([(pk[p, :rows * D].reshape(rows, D), pk[p, rows * D:])
                                       for p in range(world)])
    assert np.max(np.abs(mo.cpu().numpy() - want_o)) < 1e-5
    assert np.max(np.abs(ml.cpu().numpy() - want_l)) < 1e-5


@pytest.mark.parametrize("world", [2, 4, 8])
def test_peer_combine_emulated_ranks(cuda_handle, world):
    """ep_splitkv_combine_dev with `world` ranks in one process on one GPU
    (each rank's kernel on its own stream, buffers connected by pointer):
    every rank's result equals the K5 merge of the same partials (which the
    test above pins to the oracle), over several steps so the epoch/ack
    protocol and buffer reuse are exercised."""
    import torch
    from paper_2504_11729_b200.attention import Handle
    from paper_2504_11729_b200.splitkv import PeerSplitKVCombine, SplitKVCombine
    rows, D = 96, 128
    handles = [Handle(torch.cuda.current_device()) for _ in range(world)]
    groups = PeerSplitKVCombine.local_group(world, rows, D, handles)
    streams = [torch.cuda.Stream() for _ in range(world)]
    gen = torch.Generator(device="cuda").manual_seed(7)
    for step in range(4):
        o = torch.randn((world, rows, D), device="cuda", generator=gen)
        lse = torch.randn((world, rows), device="cuda", generator=gen) * 3
        if step == 1:
            lse[0, :5] = float("-inf")  # a rank with no visible keys for some rows
        if step == 2:
            lse[:, 7] = float("-inf")   # a fully masked row
        packed = torch.cat([torch.cat([o[p].reshape(-1), lse[p]]) for p in range(world)])
        want_o, want_l = SplitKVCombine(world, rows, D, handle=cuda_handle, device="cuda",
                                        gather=lambda out, inp: out.copy_(packed))(o[0], lse[0])
        outs = []
        torch.cuda.synchronize()
        for r in range(world):
            with torch.cuda.stream(streams[r]):
                oo = torch.empty((rows, D), dtype=torch.bfloat16 if step == 3 else torch.float32,
                                 device="cuda")
                ol = torch.empty((rows,), device="cuda")
                groups[r](o[r].contiguous(), lse[r].contiguous(), out=oo, out_lse=ol,
                          stream=streams[r])
                outs.append((oo, ol))
        torch.cuda.synchronize()
        for r, (oo, ol) in enumerate(outs):
            tol = 1e-2 if step == 3 else 1e-5
            assert torch.allclose(oo.float(), want_o, atol=tol, rtol=tol), (step, r)
            fin = torch.isfinite(want_l)
            assert torch.equal(fin, torch.isfinite(ol)), (step, r)
            assert torch.allclose(ol[fin], want_l[fin], atol=1e-5), (step, r)
    for g in groups:
        g.close()


@pytest.mark.parametrize("batch", [1, 32])
def test_torchrun_config4_two_ranks(batch):
    """Config 4 at its own shape on 2 GPUs: 131072 cloud + 512 edge keys per
    request sharded over two processes, all three combines (peer-memory
    kernel over NVLink, NCCL all-gather + K5, fused into K1); rank 0 checks the merged output
    against an unsharded single-GPU run of the same batch and against the
    fp64 oracle on sampled units (tools/splitkv_bench.py --check); and the
    combine fused into the decode kernel (ep_spliced_attention_splitkv)."""
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(29533 + batch),
           os.path.join(ROOT, "tools", "splitkv_bench.py"), "--batch", str(batch), "--steps", "3",
           "--check", "--combine", "peer", "nccl", "fused"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    print(r.stdout)
    assert r.stdout.count('"check_ok": true') == 3, r.stdout


_FUSED_EMULATED = r"""
import os, sys
sys.path.insert(0, {root!r}); sys.path.insert(0, os.path.join({root!r}, "tools"))
import torch
import splitkv_bench as SB
from paper_2504_11729_b200.attention import Handle
from paper_2504_11729_b200.splitkv import PeerSplitKVCombine
world, batch, cloud, edge = {world}, 3, 8192, 200
rows, D, HQ = batch * SB.HQ, SB.D, SB.HQ
handles = [Handle(0) for _ in range(world)]
groups = PeerSplitKVCombine.local_group(world, rows, D, handles)
ranks = [SB.build_local(batch, world, r, handles[r], cloud=cloud, edge=edge) for r in range(world)]
_, _, attn1, q1, _ = SB.build_local(batch, 1, 0, handles[0], cloud=cloud, edge=edge)
want_o, want_l = attn1(q1, o_dtype=torch.float32)
streams = [torch.cuda.Stream() for _ in range(world)]
torch.cuda.synchronize()
for step in range(4):
    outs = []
    for r in range(world):
        _, _, attn, q, _ = ranks[r]
        dt = torch.bfloat16 if step == 3 else torch.float32
        o = torch.full(q.shape, float("nan"), dtype=dt, device="cuda")
        l = torch.full(tuple(q.shape[:3]), float("nan"), device="cuda")
        groups[r].attend(attn, q, out=o, out_lse=l, stream=streams[r])
        outs.append((o, l))
    torch.cuda.synchronize()
    for r, (o, l) in enumerate(outs):
        tol = 2e-2 if step == 3 else 1e-4
        err = (o.float() - want_o).abs().max().item()
        lerr = (l - want_l).abs().max().item()
        assert err < tol and lerr < 1e-4, (step, r, err, lerr)
        assert torch.equal(o, outs[0][0]) and torch.equal(l, outs[0][1]), (step, r)  # identical on every rank
    print("step", step, "ok", err, lerr)
for g in groups:
    g.close()
print("FUSED_OK")
"""


@pytest.mark.parametrize("world", [2, 4])
def test_fused_splitkv_emulated_ranks(world):
    """ep_spliced_attention_splitkv (K1 with the cross-rank exchange fused in)
    with `world` ranks emulated on one GPU — each rank's plan on 148 / world
    SMs (EP_K1_CTAS) so all ranks' kernels run side by side, one stream each:
    every rank's merged rows equal the unsharded run (and each other,
    bit-identically), over 4 steps (epoch parity, buffer reuse, bf16 out)."""
    env = dict(os.environ, EP_K1_CTAS=str(148 // world))
    code = _FUSED_EMULATED.format(root=ROOT, world=world)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0 and "FUSED_OK" in r.stdout, r.stdout + r.stderr[-3000:]
