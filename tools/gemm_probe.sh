P=tools/gemm_probe
for v in 0 4 5; do for tn in 32 64 128 256; do $P 128 $tn 16384 $tn 3 2 $v; done; done
