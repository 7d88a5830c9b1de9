timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale_parity.py -m gpu -q -x -k "c4 or straggler or c3_1024 or c1 or irregular" > gpurun_out/s5_test.log 2>&1; echo rc=$? >> gpurun_out/s5_test.log
for i in 1 2; do timeout 300 python bench.py --config c4 --steps 5 --warmup 3 > gpurun_out/s5_c4_$i.json 2>/dev/null; done
timeout 300 python bench.py --config c3 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s5_c3_stage.json 2>/dev/null
STG_EXP_NOSTAGE=1 timeout 300 python bench.py --config c3 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s5_c3_nostage.json 2>/dev/null
C="python bench.py --config c3 --steps 1 --warmup 2 --no-e2e --no-cpu-baseline"
$C > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_sym_agg -s 2 -c 1 -o gpurun_out/s5_c3_stage $C > gpurun_out/s5_ncu.log 2>&1
