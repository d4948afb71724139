#!/bin/bash
# Device apply time (L2 flushed) of a spread of element-kernel variants,
# optionally for several library builds: tools/v2_sweep.sh [lib.so ...]
CASES=(
"32 3 cnh none 64 0" "32 3 cnh none 64 0.05" "32 3 cnh scalar 64 0" "32 3 cnh tensor 64 0" "32 3 cnh cachedF 64 0"
"32 3 inh none 64 0.05" "32 3 inh scalar 64 0.05" "32 3 inh tensor 64 0.05"
"32 3 fiber none 64 0.05" "32 3 fiber scalar 64 0.05" "32 3 fiber tensor 64 0.05"
"32 3 cnh none 64 0 spatial" "32 3 cnh tensor 64 0 spatial" "32 3 inh none 64 0.05 spatial"
"32 3 cnh none 32 0" "32 3 cnh scalar 32 0" "32 3 cnh tensor 32 0" "32 3 inh none 32 0.05" "32 3 fiber tensor 32 0.05"
"24 4 cnh none 64 0" "24 4 inh none 64 0.1" "24 4 inh tensor 64 0.1" "24 4 inh none 32 0" "24 4 inh none 32 0.1"
"32 2 cnh none 64 0" "32 2 inh none 64 0.05" "32 2 cnh none 32 0" "48 1 cnh none 64 0" "48 1 inh none 32 0")
LIBS=("$@"); [ ${#LIBS[@]} -eq 0 ] && LIBS=("")
for L in "${LIBS[@]}"; do
  echo "lib: ${L:-default}"
  for c in "${CASES[@]}"; do
    if [ -n "$L" ]; then EMFGPU_LIB=$L timeout 120 python tools/apply_ab.py $c 2>&1 | tail -1
    else timeout 120 python tools/apply_ab.py $c 2>&1 | tail -1; fi
  done
done
