#!/bin/bash
# Alternating A/B of library builds (tools/build_variant.sh) on apply_ab.py
# cases, each case in its own process, the whole list repeated REPS times:
# CASES="32 3 cnh none 64 0;24 4 inh none 64 0.1" REPS=2 tools/ab_libs.sh lib1.so lib2.so
IFS=';' read -ra CS <<< "${CASES:-32 3 cnh none 64 0}"
for rep in $(seq 1 ${REPS:-2}); do
  for L in "$@"; do
    echo "lib: $L rep $rep"
    for c in "${CS[@]}"; do EMFGPU_LIB=$L timeout 120 python tools/apply_ab.py $c 2>&1 | tail -1; done
  done
done
