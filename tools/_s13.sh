timeout 1200 python -m pytest tests -m gpu -q -x -k "not test_c4_full and not two_gpu and not sharded" > gpurun_out/s13_test.log 2>&1; echo rc=$? >> gpurun_out/s13_test.log
timeout 300 python bench.py --config c3 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s13_c3.json 2>/dev/null
C="python bench.py --config c3 --steps 1 --warmup 2 --no-e2e --no-cpu-baseline"
$C > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_sym_agg -s 2 -c 1 -o gpurun_out/s13_c3_gcoop $C > gpurun_out/s13_ncu.log 2>&1
