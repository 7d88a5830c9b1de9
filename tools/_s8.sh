timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale_parity.py tests/test_gpu_errors.py -m gpu -q -x -k "c4 or coll or straggler or irregular or c3_1024" > gpurun_out/s8_test.log 2>&1; echo rc=$? >> gpurun_out/s8_test.log
timeout 900 python -m pytest tests/test_dist.py -m gpu -q -x > gpurun_out/s8_dist.log 2>&1; echo rc=$? >> gpurun_out/s8_dist.log
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 300 python bench.py --config c4 --steps 5 --warmup 3 > gpurun_out/s8_c4_1.json 2>/dev/null
timeout 300 $R --nproc-per-node 2 --master-port 29511 bench.py --config c4 --gpus 2 --steps 5 --warmup 3 > gpurun_out/s8_c4_2.json 2>/dev/null
STG_TRACE=1 timeout 400 $R --nproc-per-node 2 --master-port 29502 bench.py --gpus 2 --steps 2 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/s8_c2_2.json 2> gpurun_out/s8_c2_2_trace.err
STG_TRACE=1 timeout 400 python bench.py --steps 2 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/s8_c2_1.json 2> gpurun_out/s8_c2_1_trace.err
STG_TRACE=1 timeout 300 $R --nproc-per-node 2 --master-port 29522 bench.py --config c3 --gpus 2 --steps 2 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/s8_c3_2.json 2> gpurun_out/s8_c3_2_trace.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s8_c4_launches.csv python bench.py --config c4 --steps 1 --warmup 1 > /dev/null 2>&1
