# 4-GPU checks of the committed head: the sharded / distributed tests (incl. the 4-GPU cases) and the
# scaling lines.  usage: gpurun --gpus 4 -- bash tools/gpu_validate4.sh   (outputs in gpurun_out/s23_*)
timeout 900 python -m pytest tests/test_dist.py -m gpu -q -x > gpurun_out/s23_dist.log 2>&1; echo rc=$? >> gpurun_out/s23_dist.log
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 400 $R --nproc-per-node 4 --master-port 29504 bench.py --gpus 4 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s23_c2_4.json 2>/dev/null
timeout 400 $R --nproc-per-node 2 --master-port 29502 bench.py --gpus 2 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s23_c2_2.json 2>/dev/null
timeout 400 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s23_c2_1.json 2>/dev/null
timeout 300 $R --nproc-per-node 4 --master-port 29524 bench.py --config c3 --gpus 4 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s23_c3_4.json 2>/dev/null
timeout 300 $R --nproc-per-node 4 --master-port 29514 bench.py --config c4 --gpus 4 --steps 5 --warmup 3 > gpurun_out/s23_c4_4.json 2>/dev/null
