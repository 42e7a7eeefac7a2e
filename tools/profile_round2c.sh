#!/bin/bash
# Round-2 (third session) profile refresh on one B200: bench lines of every
# BASELINE config (config 4 = RK4 on moving particles, the headline), the
# reference arm, per-part emulation at C4 and C5 (subtree lists on restricted
# calls), the CUPTI timeline of two RK4 steps, the subtree-vs-global list
# check, the ncu launch list of the headline command and one ncu --set full
# capture of the hot kernels. Raw outputs in gpurun_out/prof2c/ (summarised
# into profiles/r2c/).
P=${1:-gpurun_out/prof2c}
mkdir -p $P
nvidia-smi -q -d CLOCK,POWER > $P/smi.txt 2>&1
python bench.py --steps 20 --warmup 5 > $P/bench_config4.json 2> $P/c4.err
for c in c4eval c1 c2 c2pc c2log c3 c5; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 > $P/bench_$c.json 2> $P/$c.err; done
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $P/bench_reference_arm.json 2> $P/ref.err
timeout 600 python tools/timeline.py 2 --json $P/timeline_config4.json > $P/timeline_config4.txt 2>&1
timeout 600 python tools/timeline.py 1 --config c5 --json $P/timeline_config5.json > $P/timeline_config5.txt 2>&1
timeout 900 python tools/part_bench.py 1 2 4 8 --shard-bin --phases > $P/parts_config4.jsonl 2>&1
timeout 900 python tools/part_bench.py 1 2 4 8 --shard-bin --phases --config c5 > $P/parts_config5.jsonl 2>&1
SSUM_TRACE=1 timeout 600 python tools/sub_check.py l5 l7 c2 c4 c3s > $P/sub_check.txt 2>&1
# under ncu every launch is serialised and slowed, so the measured list-builder
# choice would pick the one-launch subtree builder; pin the builder the live
# bench uses at this size (the global traversal, see timeline_config4.txt)
SSUM_SUB_LISTS=0 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $P/launches_config4.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-error > $P/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_tiles|k_finish|k_up_partial|k_walk|k_bfs|k_leaf_fill|k_rk4|k_sub_lists" -c 12 -o $P/full python tools/profile_step.py 1 > $P/ncu_full.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_tiles" -c 2 -o $P/full_log python tools/profile_step.py 1 8 8 0.7 log > $P/ncu_full_log.log 2>&1
timeout 600 python tools/host_overhead.py 4 > $P/host_overhead.txt 2>&1
ls -la $P
