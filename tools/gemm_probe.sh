# tcgen05 issue probe (tools/gemm_probe.cu): one CTA, K = 16384 (256 k-blocks of 64), clock64 per k-block
# args: rows vocab K tn stages mode variant   (mode 0 full / 1 TMA only / 2 MMA only; variant 0 one accumulator,
#       1 two N/2 MMAs into two accumulators, 3 alternate accumulators per K16 step, 4 A from TMEM, 5 M = 64)
P=tools/gemm_probe
for v in 0 4 5; do for tn in 32 64 128 256; do $P 128 $tn 16384 $tn 3 2 $v; done; done
for v in 1 3; do $P 128 256 16384 256 3 2 $v; done
for m in 1 0; do $P 128 256 16384 256 3 $m 0; done
$P 576 4096 4096 256 4 0 0
$P 576 4096 4096 160 5 0 0
