# 4-GPU validation: sharded stage d tests at 2 and 4 GPUs, scaling lines
timeout 1200 python -m pytest tests/test_dist.py -m gpu -q -x > gpurun_out/s7_dist.log 2>&1; echo rc=$? >> gpurun_out/s7_dist.log
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for n in 2 4; do
  timeout 400 $R --nproc-per-node $n --master-port 2950$n bench.py --gpus $n --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s7_c2_$n.json 2> gpurun_out/s7_c2_$n.err
  timeout 300 $R --nproc-per-node $n --master-port 2951$n bench.py --config c4 --gpus $n --steps 5 --warmup 3 > gpurun_out/s7_c4_$n.json 2> gpurun_out/s7_c4_$n.err
  timeout 300 $R --nproc-per-node $n --master-port 2952$n bench.py --config c3 --gpus $n --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s7_c3_$n.json 2> gpurun_out/s7_c3_$n.err
done
timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s7_c2_1.json 2> gpurun_out/s7_c2_1.err
