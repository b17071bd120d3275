import json, sys, torch
sys.path.insert(0, '.')
from paper_2504_11729_b200 import model as M
g = json.load(open('tests/golden/model_golden.json'))
m = M.Model(M.ModelConfig(2, 4, 256, 256, 1024, 42), dtype="f32", kv_dtype="f32", num_pages=128)
c = M.SegmentedCache(m)
p = M.prefill(m, g['cfg1_cloud'], M.ORIGIN_CLOUD, 0, c); c.append(p.segments)
e = M.prefill(m, g['cfg1_edge'], M.ORIGIN_EDGE, 512, c); c.append(e.segments)
M.generate_batch(m, [c], [e.next_token], 3)
torch.cuda.synchronize()
