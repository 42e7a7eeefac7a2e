#!/bin/bash
# Round profile refresh (one B200): bench lines of every BASELINE config, the
# per-part and RK4 timings, the ncu launch list and one ncu --set full
# capture of the hot kernels, all under gpurun_out/prof/ (then summarised
# into profiles/ by tools/summarize_profiles.py).
mkdir -p gpurun_out/prof
python bench.py --steps 10 --warmup 3 > gpurun_out/prof/r1_bench_config4.json 2> gpurun_out/prof/c4.err
for c in c2 c2pc c2log c3 c5; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/prof/r1_bench_$c.json 2> gpurun_out/prof/$c.err; done
timeout 600 python tools/part_bench.py 1 2 4 8 --phases > gpurun_out/prof/r1_parts_config4.jsonl 2>&1
timeout 600 python tools/rk4_bench.py --steps 49 --reference > gpurun_out/prof/r1_rk4_config4.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/r1_launches_config4.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-error > gpurun_out/prof/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_tiles|k_finish|k_up_partial|k_walk|k_bfs|k_leaf_fill" -c 8 -o gpurun_out/prof/full python tools/profile_step.py 1 > gpurun_out/prof/ncu_full.log 2>&1
ls -la gpurun_out/prof
