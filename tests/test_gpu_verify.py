"""GPU parity of K3 (tcgen05 multi-row verify attention): n_q = k+1 causal
rows per request (k = 4, 8) with GQA group 4 -> 20 / 36 rows per kv-head,
against the fp64 oracle on identical bf16 inputs (2e-2 relative, north_star)."""
import os
import subprocess
import sys

import numpy as np
import pytest

from oracle import oracle as O
from tests import splice_cases as SC
from tests.gpu_util import to_device
from tests.test_gpu_decode import _check

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("k", [4, 8])
def test_config3_shape_subset(cuda_handle, k):
    """BASELINE config 3 structure (cloud 14336 + edge 1536 + generated 512
    = 16384 keys, drafts causal at the end) at batch 4, checked on 24 units."""
    reqs = [[(SC.CLOUD, 14336, None), (SC.EDGE, 1536, None), (SC.GEN, 512, None)]] * 4
    sb = SC.make_case(O.DT_BF16, 32, 8, 128, reqs, n_q=k + 1, seed=31)
    _, _, attn, q = to_device(sb, cuda_handle)
    o, lse = attn(q)
    units = np.random.default_rng(k).choice(4 * 32, 24, replace=False)
    want_o, want_l = O.spliced_attention(sb, n_threads=os.cpu_count() or 4, units=units)
    print(f"cfg3 k={k} rel err:", _check(o, lse, want_o, want_l, sb.kv_dtype, units, 32))


def test_tc_path_on_decode_rows_matches_golden():
    """EP_FORCE_TC=1 routes a 4-row decode through the tcgen05 kernel: it must
    reproduce the reference goldens like the CUDA-core kernel does."""
    code = (
        "import numpy as np, os, sys; sys.path.insert(0, %r)\n"
        "from tests import splice_cases as SC\n"
        "from tests.gpu_util import to_device\n"
        "from tests.cases import rel_err\n"
        "g = np.load(os.path.join(%r, 'tests/golden/splice_golden.npz'))\n"
        "for name in ['gqa4_bf16_decode', 'gqa2_f32_d128_nq2']:\n"
        "    sb = SC.small_case(name)\n"
        "    if sb.kv_dtype != 1: continue\n"
        "    _, _, attn, q = to_device(sb)\n"
        "    import torch\n"
        "    o, l = attn(q, o_dtype=torch.float32)\n"
        "    e = rel_err(o.cpu().numpy(), g[name + '/out'])\n"
        "    assert e <= 2e-2, (name, e)\n"
        "    print(name, e)\n" % (ROOT, ROOT))
    env = dict(os.environ, EP_FORCE_TC="1")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    print(r.stdout)
