"""GPU parity of the cross-GPU split-KV path (config 4).

* On one GPU: P "ranks" are emulated as P shard plans over separate pools;
  their fp32 (o, lse) partials are packed exactly as the NCCL all-gather packs
  them and merged by the K5 kernel — compared with the unsharded spliced
  attention and with the fp64 oracle.
* With >= 2 GPUs: tools/splitkv_bench.py --check under torchrun (NCCL
  all-gather across real ranks, merged result checked against an unsharded
  single-GPU run)."""
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


def test_torchrun_nccl_two_ranks():
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29533",
           os.path.join(ROOT, "tools", "splitkv_bench.py"), "--batch", "2", "--steps", "3",
           "--check"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    assert '"check_ok": true' in r.stdout, r.stdout
