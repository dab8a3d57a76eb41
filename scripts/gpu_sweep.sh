#!/bin/bash
# tuning sweep of the fused kernel: library variant x tile size x stage count (cfg2, 40 iterations)
mkdir -p gpurun_out
out=gpurun_out/sweep.txt; : > $out
run() {  # lib tps nbuf
  r=$(PF_B200_LIB=$1 PF_FAST_TPS=$2 PF_FAST_NBUF=$3 timeout 300 python scripts/prof_fused.py cfg2 40 2>&1 | tail -1)
  echo "lib=$1 tps=$2 nbuf=$3 :: $r" | tee -a $out
}
B=paper_2605_01748_b200/_build
for a in ${SWEEP:-"libpf_b200.so 2048 1"}; do :; done
while read lib tps nbuf; do [ -n "$lib" ] && run $B/$lib $tps $nbuf; done <<< "$SWEEP"
