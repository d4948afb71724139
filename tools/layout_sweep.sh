#!/bin/bash
# Rebuild the Q3 element kernels for several padded layouts (SZ, SIZE) of
# Lay<4> and time cfg1 with bench.py (element phase per variant).
# usage: tools/layout_sweep.sh "SZ:SIZE ..."   (run on the GPU box)
set -e
CS=paper_2408_12479_b200/csrc
cp $CS/apply_v2.cuh /tmp/apply_v2.cuh.orig
for cfg in $1; do
  SZ=${cfg%%:*}; SIZE=${cfg##*:}
  sed -i "s/struct Lay<4> { static constexpr int N = 4, N2 = 16, N3 = 64, SY = 4, SZ = [0-9]*, SIZE = [0-9]*; };/struct Lay<4> { static constexpr int N = 4, N2 = 16, N3 = 64, SY = 4, SZ = $SZ, SIZE = $SIZE; };/" $CS/apply_v2.cuh
  make -s -C $CS -j8 > /tmp/lay_make.log 2>&1 || { echo "build failed $cfg"; tail -3 /tmp/lay_make.log; continue; }
  python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-extra 2>/dev/null | tail -1 > gpurun_out/lay_$SZ_$SIZE.json
  python -c "
import json,sys
d=json.loads(open('gpurun_out/lay_$SZ_$SIZE.json').read())
v=d['variants']
print('SZ=$SZ SIZE=$SIZE', ' '.join('%s=%.4f'%(k,v[k]['ms_element_kernel']) for k in ('fp64_none','fp64_scalar','fp64_tensor','fp32_none','fp32_tensor','fp64_spatial_none')))
"
done
cp /tmp/apply_v2.cuh.orig $CS/apply_v2.cuh
