#!/bin/bash
# Layout sweep for Lay<5> (Q4): "SY:SZ:SIZE ..."; times 32^3 Q4 curved iNH (cfg2-like) fp64/fp32 none and fp64 tensor.
set -e
CS=paper_2408_12479_b200/csrc
cp $CS/apply_v2.cuh /tmp/apply_v2.cuh.orig
for cfg in $1; do
  IFS=: read SY SZ SIZE <<< "$cfg"
  sed -i "s/struct Lay<5> { static constexpr int N = 5, N2 = 25, N3 = 125, SY = [0-9]*, SZ = [0-9]*, SIZE = [0-9]*; };/struct Lay<5> { static constexpr int N = 5, N2 = 25, N3 = 125, SY = $SY, SZ = $SZ, SIZE = $SIZE; };/" $CS/apply_v2.cuh
  make -s -C $CS -j8 > /tmp/lay_make.log 2>&1 || { echo "build failed $cfg"; tail -3 /tmp/lay_make.log; continue; }
  echo "== SY=$SY SZ=$SZ SIZE=$SIZE"
  python tools/time_apply.py 32 4 inh none 64 0.1
  python tools/time_apply.py 32 4 inh none 32 0.1
  python tools/time_apply.py 32 4 inh tensor 64 0.1
done
cp /tmp/apply_v2.cuh.orig $CS/apply_v2.cuh
