python -m pytest tests -m gpu -x -q > gpurun_out/r02_gputest_loc.log 2>&1; tail -2 gpurun_out/r02_gputest_loc.log
for r in 1 2; do for L in libemfgpu var_locold; do
  EMFGPU_LIB=paper_2408_12479_b200/lib/$L.so timeout 300 python tools/cfg2_time.py 64:none 64:tensor 32:none 2>&1 | grep -v Warn
  EMFGPU_LIB=paper_2408_12479_b200/lib/$L.so timeout 300 python tools/apply_ab.py 32 3 cnh none 64 0 2>&1 | tail -1
  EMFGPU_LIB=paper_2408_12479_b200/lib/$L.so timeout 300 python tools/apply_ab.py 32 3 cnh none 32 0 2>&1 | tail -1
done; done > gpurun_out/r02_loc.txt 2>&1; cat gpurun_out/r02_loc.txt
