# K9 persistent rollout: tests, rollout timing vs the graph path, barrier trace
timeout 300 python -m pytest tests/test_gpu_model.py -q -x 2>&1 | tail -2
for c in ${K9_CTAS:-148}; do
  EP_PERSIST_CTAS=$c EP_MODEL_PERSIST=1 timeout 300 python tools/model_bench.py --batch 8 --steps 32 > gpurun_out/mb_1_$c.json 2>&1
  EP_PERSIST_CTAS=$c EP_MODEL_PERSIST=1 EP_TRACE=1 EP_TRACE_FILE=gpurun_out/trace_persist_$c.bin timeout 120 python tools/prof_model_rollout.py
done
EP_MODEL_PERSIST=0 timeout 300 python tools/model_bench.py --batch 8 --steps 32 > gpurun_out/mb_0.json 2>&1
