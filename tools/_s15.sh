for g in 64 128 256 96 48 64; do
STG_EXP_GRID=$g timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s15_c2_g$g.json 2>/dev/null
done
for g in 128 256; do
STG_EXP_GRID=$g timeout 300 python bench.py --config c3 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s15_c3_g$g.json 2>/dev/null
done
