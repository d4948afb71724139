python tools/cfg2_time.py 32:none > gpurun_out/plain1.log 2>&1 && python tools/time_apply.py 32 3 cnh none 32 > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:apply_v2_kernel -s 3 -c 1 -o gpurun_out/r02_f32_q4 python tools/cfg2_time.py 32:none > gpurun_out/ncu1.log 2>&1; \
ncu --set full --clock-control none --import-source on -k regex:apply_v3_kernel -s 3 -c 1 -o gpurun_out/r02_f32_q3 python tools/time_apply.py 32 3 cnh none 32 > gpurun_out/ncu2.log 2>&1; \
cat gpurun_out/plain1.log gpurun_out/plain2.log
