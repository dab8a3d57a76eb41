#!/bin/bash
# tile-phase clock64 probe (variant build _build/tprobe, -DPF_TPROBE): cycles per tile by phase
for c in ${CFGS:-cfg2}; do
  PF_B200_LIB=paper_2605_01748_b200/_build/tprobe/libpf_b200.so python scripts/prof_fused_warm.py $c 100 100 2>&1 | tail -3
done
