# Full GPU validation of the committed head on a 2-GPU box: pytest -m gpu (incl. the 2-GPU tests), smoke, the driver's bench lines.
# usage: gpurun --gpus 2 -- bash tools/gpu_validate.sh   (outputs in gpurun_out/s22_*)
timeout 1800 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/s22_gputest.log 2>&1; echo rc=$? >> gpurun_out/s22_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s22_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/s22_bench.json 2> gpurun_out/s22_bench.err
timeout 400 python bench.py --config c3 --steps 5 --warmup 3 > gpurun_out/s22_c3.json 2> gpurun_out/s22_c3.err
timeout 300 python bench.py --config c4 --steps 5 --warmup 3 > gpurun_out/s22_c4.json 2> gpurun_out/s22_c4.err
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 $R --nproc-per-node 2 --master-port 29502 bench.py --gpus 2 > gpurun_out/s22_c2_2.json 2> gpurun_out/s22_c2_2.err
