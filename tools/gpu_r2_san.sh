set -x
mkdir -p gpurun_out/r2san
python tools/sanitize_step.py > gpurun_out/r2san/plain.log 2>&1; echo plain_rc=$?
timeout 900 compute-sanitizer --tool racecheck --racecheck-report analysis python tools/sanitize_step.py > gpurun_out/r2san/racecheck.log 2>&1; echo race_rc=$?
timeout 900 compute-sanitizer --tool synccheck python tools/sanitize_step.py > gpurun_out/r2san/synccheck.log 2>&1; echo sync_rc=$?
timeout 900 compute-sanitizer --tool memcheck python tools/sanitize_step.py > gpurun_out/r2san/memcheck.log 2>&1; echo mem_rc=$?
SSUM_TRACE=1 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-error > gpurun_out/b3.json 2> gpurun_out/b3.err; echo bench_rc=$?
tail -3 gpurun_out/r2san/*.log
