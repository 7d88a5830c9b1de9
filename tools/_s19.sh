timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/s19_gputest.log 2>&1; echo rc=$? >> gpurun_out/s19_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s19_smoke.log 2>&1
timeout 400 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s19_c2.json 2>/dev/null
timeout 400 python bench.py --config c3 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s19_c3.json 2>/dev/null
STG_TRACE=1 timeout 400 python bench.py --config c3 --steps 1 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/s19_c3_trace.json 2> gpurun_out/s19_c3_trace.err
timeout 300 python bench.py --config c4 --steps 5 --warmup 3 > gpurun_out/s19_c4.json 2>/dev/null
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
STG_TRACE=1 timeout 400 $R --nproc-per-node 2 --master-port 29502 bench.py --gpus 2 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s19_c2_2.json 2> gpurun_out/s19_c2_2_trace.err
