"""Decoder on the GPU at BASELINE config 1: the reference
tiny decoder (L=2, H=4, d_model=256, d_head=64, V=256, seed 42, fp32) over a
512-token cloud segment + 64-token edge segment (the golden prompts), greedy.

  * decode_step latency, batch 1, through the public API (host token in,
    host token out every step = the reference's decode_step contract), and
    the device time of the same forward pass (CUDA events);
  * batched decode: B sessions sharing the cloud prompt's pages, one forward
    per step (tokens/s);
  * cloud + edge prefill latency;
  * the reference's own decode_step / prefill (oracle/_ref, fp64, one host
    thread — the function is sequential) on the same prompts.

    python tools/model_bench.py [--steps 64] [--warmup 5]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CFG1 = (2, 4, 256, 256, 1024, 42)


def _prompts():
    with open(os.path.join(ROOT, "tests", "golden", "model_golden.json")) as f:
        g = json.load(f)
    return g["cfg1_cloud"], g["cfg1_edge"]


def run(steps: int, warmup: int, h=None, batch: int = 64, cpu: bool = True):
    import torch
    from paper_2504_11729_b200 import model as M
    cloud, edge = _prompts()
    m = M.Model(M.ModelConfig(*CFG1), dtype="f32", kv_dtype="f32", handle=h,
                num_pages=(batch + 2) * 24 + 64)
    out = {"workload": "cfg1 tiny decoder L=2 H=4 d_model=256 V=256 fp32, cloud 512 + edge 64, "
                       "greedy decode"}

    # ---- prefill latency (cloud then edge), device events ----
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    times = []
    for it in range(warmup + 5):
        cache = M.SegmentedCache(m)
        torch.cuda.synchronize()
        ev[0].record()
        pc = M.prefill(m, cloud, M.ORIGIN_CLOUD, 0, cache, want_hidden=False)
        cache.append(pc.segments)
        ev[1].record()
        pe = M.prefill(m, edge, M.ORIGIN_EDGE, len(cloud), cache, want_hidden=False)
        cache.append(pe.segments)
        ev[2].record()
        torch.cuda.synchronize()
        if it >= warmup:
            times.append((ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2])))
        if it < warmup + 4:
            cache.release()
    out["prefill_ms"] = {"cloud512": statistics.median(t[0] for t in times),
                         "edge64": statistics.median(t[1] for t in times)}

    # ---- batch-1 decode through the public API (token round trip per step) ----
    tok = pe.next_token
    for _ in range(warmup):
        tok = M.decode_step(m, cache, tok).next_token
    torch.cuda.synchronize()
    lat = []
    for _ in range(steps):
        t0 = time.perf_counter()
        nxt, _ = M.decode_batch(m, [cache], [tok])
        tok = int(nxt[0])
        lat.append((time.perf_counter() - t0) * 1e3)
    # device time of the forward alone
    dev = []
    for _ in range(steps // 2):
        cache._grow_generated(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        nx, _, _ = m.forward([cache.segments], [1], [tok], want_logits=False)
        e1.record()
        torch.cuda.synchronize()
        tok = int(nx[0].item())
        dev.append(e0.elapsed_time(e1))
    l0 = m.handle.launch_count()
    M.decode_batch(m, [cache], [tok])
    out["decode_b1"] = {"api_ms_p50": statistics.median(lat), "api_ms_p99": sorted(lat)[int(0.99 * (len(lat) - 1))],
                        "device_ms_p50": statistics.median(dev), "launches_per_step": m.handle.launch_count() - l0,
                        "attention_path": m.last_attention_path(), "end_position": cache.end_position()}
    cache.release()

    # ---- device-resident rollout (ep_model_generate: one CUDA graph per step) ----
    roll = {}
    for nb in (1, batch):
        base = M.SegmentedCache(m)
        pc = M.prefill(m, cloud, M.ORIGIN_CLOUD, 0, base, want_hidden=False)
        caches, toks = [], []
        for b in range(nb):
            c = M.SegmentedCache(m)
            m.pages.retain(pc.segment.pages)
            c.append(pc.segments)
            e = M.prefill(m, edge, M.ORIGIN_EDGE, len(cloud), c, want_hidden=False)
            c.append(e.segments)
            caches.append(c)
            toks.append(e.next_token)
        M.generate_batch(m, caches, toks, 4)  # warm-up (graph build paths, plan buffers)
        torch.cuda.synchronize()
        n_roll = 256
        t0 = time.perf_counter()
        out_t = M.generate_batch(m, caches, toks, n_roll)
        el = time.perf_counter() - t0
        roll[f"b{nb}"] = {"steps": n_roll, "ms_per_step": el / n_roll * 1e3,
                          "tokens_per_s": nb * n_roll / el, "attention_path": m.last_attention_path()}
        for c in caches:
            c.release()
        base.release()
        del out_t
    out["rollout_device"] = roll

    # ---- batched decode: B sessions share the cloud prompt ----
    base = M.SegmentedCache(m)
    pc = M.prefill(m, cloud, M.ORIGIN_CLOUD, 0, base, want_hidden=False)
    caches, toks = [], []
    for b in range(batch):
        c = M.SegmentedCache(m)
        m.pages.retain(pc.segment.pages)
        c.append(pc.segments)
        e = M.prefill(m, edge, M.ORIGIN_EDGE, len(cloud), c, want_hidden=False)
        c.append(e.segments)
        caches.append(c)
        toks.append(e.next_token)
    for _ in range(warmup):
        nxt, _ = M.decode_batch(m, caches, toks)
        toks = [int(t) for t in nxt]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    n_b = max(8, steps // 4)
    for _ in range(n_b):
        nxt, _ = M.decode_batch(m, caches, toks)
        toks = [int(t) for t in nxt]
    el = time.perf_counter() - t0
    out[f"decode_b{batch}"] = {"api_ms_per_step": el / n_b * 1e3, "tokens_per_s": batch * n_b / el,
                               "attention_path": m.last_attention_path()}
    for c in caches:
        c.release()

    if cpu:
        from oracle import oracle as O
        if O.available("ref"):
            t0 = time.perf_counter()
            ses = O.RefModel(*CFG1).session(cloud, edge)
            t_pre = time.perf_counter() - t0
            tok = ses.first_token()
            lat = []
            for _ in range(min(steps, 16)):
                t0 = time.perf_counter()
                tok, _ = ses.decode_step(tok)
                lat.append((time.perf_counter() - t0) * 1e3)
            out["reference_cpu"] = {"decode_ms_p50": statistics.median(lat),
                                    "cloud_edge_prefill_ms": t_pre * 1e3, "threads": 1,
                                    "kind": "reference (oracle/_ref, unmodified sources, fp64)"}
            out["speedup_decode_api_vs_reference"] = (out["reference_cpu"]["decode_ms_p50"] /
                                                      out["decode_b1"]["api_ms_p50"])
            out["speedup_rollout_b1_vs_reference"] = (out["reference_cpu"]["decode_ms_p50"] /
                                                      roll["b1"]["ms_per_step"])
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=64)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--batch", type=int, default=64)
    a = ap.parse_args()
    print(json.dumps(run(a.steps, a.warmup, batch=a.batch), indent=1))


if __name__ == "__main__":
    main()
