timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/s6_test.log 2>&1; echo rc=$? >> gpurun_out/s6_test.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s6_c2.json 2>/dev/null
timeout 300 python bench.py --config c3 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s6_c3.json 2>/dev/null
timeout 300 python bench.py --config c4 --steps 5 --warmup 3 > gpurun_out/s6_c4.json 2>/dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s6_c4_launches.csv python bench.py --config c4 --steps 1 --warmup 1 > /dev/null 2>&1
