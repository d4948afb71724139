for L in libemfgpu var_q4cart4 var_q3all4 var_symall; do
  EMFGPU_LIB=paper_2408_12479_b200/lib/$L.so timeout 300 python tools/cfg2_time.py 64:none 64:scalar 64:cachedF 64:tensor 32:none 2>&1 | grep -v Warn
done > gpurun_out/r02_sym_cfg2.txt 2>&1
bash tools/v2_sweep.sh paper_2408_12479_b200/lib/libemfgpu.so paper_2408_12479_b200/lib/var_q4cart4.so paper_2408_12479_b200/lib/var_q3all4.so paper_2408_12479_b200/lib/var_symall.so > gpurun_out/r02_sym_sweep.txt 2>&1
python -m pytest tests -m gpu -x -q > gpurun_out/r02_gputest_sym.log 2>&1
tail -2 gpurun_out/r02_gputest_sym.log
