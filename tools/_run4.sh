for L in libemfgpu var_nomap; do
  EMFGPU_LIB=paper_2408_12479_b200/lib/$L.so timeout 300 python tools/cfg2_time.py 64:none 64:scalar 64:cachedF 64:tensor 2>&1 | grep -v Warn
done > gpurun_out/r02_map_cfg2.txt 2>&1
python -m pytest tests -m gpu -x -q > gpurun_out/r02_gputest_map.log 2>&1
tail -2 gpurun_out/r02_gputest_map.log
python tools/cfg2_time.py 64:none > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:apply_v2_kernel -s 3 -c 1 -o gpurun_out/r02_cfg2_map python tools/cfg2_time.py 64:none > gpurun_out/ncu.log 2>&1
