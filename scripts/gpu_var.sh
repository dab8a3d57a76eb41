#!/bin/bash
# settled timings of tuning variants: VARS="name[:ENV=V ...];..." (name 'main' = the in-tree library)
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
IFS=';' read -ra VS <<< "${VARS:-main}"
for c in ${CFGS:-cfg2}; do
  for rep in 1 2; do
    for v in "${VS[@]}"; do
      name=${v%%:*}; envs=""; [[ "$v" == *:* ]] && envs=${v#*:}
      lib=""; [ "$name" != "main" ] && lib="PF_B200_LIB=paper_2605_01748_b200/_build/$name/libpf_b200.so"
      echo "$v: $(env $lib $envs python scripts/prof_fused_warm.py $c ${W:-200} ${N:-300} 2>&1 | tail -1)"
    done
  done
done
