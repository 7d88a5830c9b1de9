# the driver's commands at N = 2 (default K/W, e2e and all): ours, then the reference arm
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 900 $R --master-port 29561 bench.py --gpus 2 > gpurun_out/s18_c2_2.json 2> gpurun_out/s18_c2_2.err; echo rc=$? >> gpurun_out/s18_c2_2.err
timeout 900 $R --master-port 29562 bench.py --impl reference --gpus 2 --steps 2 --warmup 3 > gpurun_out/s18_ref_2.json 2> gpurun_out/s18_ref_2.err; echo rc=$? >> gpurun_out/s18_ref_2.err
