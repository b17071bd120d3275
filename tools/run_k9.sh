# K9 persistent rollout vs the CUDA-graph path: model tests, rollout timing, barrier trace
[ -n "$K9_TESTS" ] && timeout 300 python -m pytest tests/test_gpu_model.py -q -x 2>&1 | tail -2
for p in ${K9_MODES:-1 0}; do
  EP_MODEL_PERSIST=$p timeout 300 python tools/model_bench.py --batch ${K9_BATCH:-4} --steps 32 > gpurun_out/mb_$p.json 2>&1
done
EP_MODEL_PERSIST=1 EP_TRACE=1 EP_TRACE_FILE=gpurun_out/trace_persist_1.bin timeout 120 python tools/prof_model_rollout.py
true
