#!/bin/bash
# Round-2 profile refresh (one B200): the bench line of every BASELINE config
# (config 4 = RK4 on moving particles, the headline), the reference arm, the
# RK4 50-step run, per-part emulation at C4 and C5, the ncu launch list of the
# headline command and one ncu --set full capture of the hot kernels inside
# an RK4 evaluation. Raw outputs land in gpurun_out/prof2/ (summarised into
# profiles/ by tools/summarize_profiles.py).
P=gpurun_out/prof2
mkdir -p $P
python bench.py --steps 20 --warmup 5 > $P/r2_bench_config4.json 2> $P/c4.err
for c in c4eval c1 c2 c2pc c2log c3 c5; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 > $P/r2_bench_$c.json 2> $P/$c.err; done
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $P/r2_bench_reference_arm.json 2> $P/ref.err
timeout 900 python tools/rk4_bench.py --steps 49 > $P/r2_rk4_config4_50steps.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $P/r2_launches_config4.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-error > $P/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_tiles|k_finish|k_up_partial|k_walk|k_bfs|k_leaf_fill|k_rk4" -c 10 -o $P/full python tools/profile_step.py 1 > $P/ncu_full.log 2>&1
ls -la $P
