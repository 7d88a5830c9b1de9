timeout 900 python -m pytest tests/test_dist.py -m gpu -q -x > gpurun_out/s17_dist.log 2>&1; echo rc=$? >> gpurun_out/s17_dist.log
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for n in 2 4; do
STG_TRACE=1 timeout 400 $R --nproc-per-node $n --master-port 2950$n bench.py --gpus $n --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s17_c2_$n.json 2> gpurun_out/s17_c2_${n}_trace.err
timeout 300 $R --nproc-per-node $n --master-port 2952$n bench.py --config c3 --gpus $n --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s17_c3_$n.json 2>/dev/null
timeout 300 $R --nproc-per-node $n --master-port 2951$n bench.py --config c4 --gpus $n --steps 5 --warmup 3 > gpurun_out/s17_c4_$n.json 2>/dev/null
done
timeout 400 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s17_c2_1.json 2>/dev/null
