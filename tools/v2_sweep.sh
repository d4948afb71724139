CASES=(
"32 3 cnh none 64 0" "32 3 cnh none 64 0.05" "32 3 cnh scalar 64 0" "32 3 inh none 64 0.05" "32 3 inh scalar 64 0.05"
"32 3 fiber none 64 0.05" "32 3 fiber scalar 64 0.05" "32 3 cnh none 64 0 spatial" "32 3 cnh tensor 64 0 spatial" "32 3 inh none 64 0.05 spatial"
"24 4 cnh none 64 0" "24 4 cnh none 64 0.1" "24 4 inh none 64 0.1" "24 4 inh tensor 64 0.1" "24 4 inh scalar 64 0.1" "24 4 cnh tensor 64 0"
"24 4 inh none 32 0.1" "32 2 cnh none 64 0" "32 2 inh none 64 0.05" "32 2 fiber none 64 0.05" "48 1 cnh none 64 0" "48 1 inh none 32 0")
for L in "" "EMFGPU_LIB=paper_2408_12479_b200/lib/var_fresh1.so"; do
  echo "lib: $L"
  for c in "${CASES[@]}"; do env $L timeout 120 python tools/apply_ab.py $c 2>&1 | tail -1; done
done
