for L in libemfgpu var_nomap32 var_f32m5 var_f32m6; do
  EMFGPU_LIB=paper_2408_12479_b200/lib/$L.so timeout 300 python tools/cfg2_time.py 32:none 32:scalar 2>&1 | grep -v Warn
  EMFGPU_LIB=paper_2408_12479_b200/lib/$L.so timeout 300 python tools/time_apply.py 24 4 inh none 32 0 2>&1 | tail -1
done > gpurun_out/r02_map32.txt 2>&1
python -m pytest tests -m gpu -x -q > gpurun_out/r02_gputest_map32.log 2>&1
tail -2 gpurun_out/r02_gputest_map32.log; cat gpurun_out/r02_map32.txt
