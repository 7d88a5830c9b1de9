# final validation of the committed head (2 GPUs: the dist tests run too)
timeout 1800 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/s16_gputest.log 2>&1; echo rc=$? >> gpurun_out/s16_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s16_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/s16_bench.json 2> gpurun_out/s16_bench.err
timeout 400 python bench.py --config c3 --steps 5 --warmup 3 > gpurun_out/s16_c3.json 2> gpurun_out/s16_c3.err
timeout 300 python bench.py --config c4 --steps 5 --warmup 3 > gpurun_out/s16_c4.json 2> gpurun_out/s16_c4.err
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 400 $R --nproc-per-node 2 --master-port 29502 bench.py --gpus 2 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s16_c2_2.json 2> gpurun_out/s16_c2_2.err
C="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
$C > /dev/null 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s16_c2_launches.csv $C > /dev/null 2>&1
$C > /dev/null 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sym_agg -s 3 -c 1 -o gpurun_out/s16_c2_ksym $C > gpurun_out/s16_ncu.log 2>&1
