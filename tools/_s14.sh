for g in 16 4 8 32 64 16; do
STG_EXP_GRID=$g timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s14_c2_g$g.json 2>/dev/null
STG_EXP_GRID=$g timeout 300 python bench.py --config c3 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s14_c3_g$g.json 2>/dev/null
done
