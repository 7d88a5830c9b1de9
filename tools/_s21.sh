for i in 1 2; do
timeout 400 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s21_c2_$i.json 2>/dev/null
timeout 400 python bench.py --config c3 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s21_c3_$i.json 2>/dev/null
done
STG_TRACE=1 timeout 400 python bench.py --config c3 --steps 1 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/s21_c3_trace.json 2> gpurun_out/s21_c3_trace.err
timeout 300 python bench.py --config c4 --steps 5 --warmup 3 > gpurun_out/s21_c4.json 2>/dev/null
