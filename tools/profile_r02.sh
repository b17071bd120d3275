# Round-2 ncu captures (one kernel each, --set full, clocks not locked), summarised
# into gpurun_out/r02_*.txt by tools/ncu_summary.py; copy the ones kept to profiles/.
set -x
N="ncu --set full --clock-control none --import-source on"
$N -k regex:spliced_decode -s 3 -c 1 -f -o gpurun_out/r02_decode python tools/decode_only.py --steps 5 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/r02_decode.ncu-rep "ncu --set full -k spliced_decode -s 3 -c 1 python tools/decode_only.py --steps 5  (K1 bf16 D=128 R=4, config 2: B=32 Hq=32 Hkv=8 4609 keys; algorithmic 603,979,776 B/launch; epilogue warp + split-first item order)" > gpurun_out/r02_decode_full.txt
$N -k regex:spliced_decode -s 2 -c 1 -f -o gpurun_out/r02_cascade_k1 python tools/multitenant_bench.py --steps 3 --warmup 1 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/r02_cascade_k1.ncu-rep "ncu --set full -k spliced_decode -s 2 -c 1 python tools/multitenant_bench.py  (config 5 private pass on K1, 123 of 148 SMs, beside the K3 shared-prefix pass)" > gpurun_out/r02_cascade_k1_full.txt
$N -k regex:verify_attention -s 2 -c 1 -f -o gpurun_out/r02_cascade_k3 python tools/multitenant_bench.py --steps 3 --warmup 1 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/r02_cascade_k3.ncu-rep "ncu --set full -k verify_attention -s 2 -c 1 python tools/multitenant_bench.py  (config 5 shared-prefix pass: K3 128-row tiles over the 8192-token cloud prompt)" > gpurun_out/r02_cascade_k3_full.txt
$N -k regex:score_argmax -s 2 -c 1 -f -o gpurun_out/r02_score python tools/verify_bench.py --k 8 --steps 3 --warmup 1 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/r02_score.ncu-rep "ncu --set full -k score_argmax -s 2 -c 1 python tools/verify_bench.py --k 8  (K4 score GEMM: 576 rows x 4096 vocab x K 4096 bf16 hi part; 19.3 GFLOP)" > gpurun_out/r02_score_full.txt
$N -k regex:verify_attention -s 2 -c 1 -f -o gpurun_out/r02_prefill python tools/prefill_bench.py --kind cloud --steps 3 --warmup 1 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/r02_prefill.ncu-rep "ncu --set full -k verify_attention -s 2 -c 1 python tools/prefill_bench.py --kind cloud  (K3 prefill tiles: 4 x 4096-token cloud prompts, causal, Hq 32 / Hkv 8, d 128 bf16)" > gpurun_out/r02_prefill_full.txt
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_bench_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
echo done
