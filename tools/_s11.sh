# final single-GPU validation of the committed head
timeout 1500 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/s11_gputest.log 2>&1; echo rc=$? >> gpurun_out/s11_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s11_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/s11_bench.json 2> gpurun_out/s11_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/s11_ref.json 2> gpurun_out/s11_ref.err
timeout 400 python bench.py --config c3 --steps 5 --warmup 3 > gpurun_out/s11_c3.json 2> gpurun_out/s11_c3.err
timeout 300 python bench.py --config c4 --steps 5 --warmup 3 > gpurun_out/s11_c4.json 2> gpurun_out/s11_c4.err
C="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
$C > /dev/null 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s11_c2_launches.csv $C > /dev/null 2>&1
$C > /dev/null 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sym_agg -s 3 -c 1 -o gpurun_out/s11_c2_ksym $C > gpurun_out/s11_ncu.log 2>&1
