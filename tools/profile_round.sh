#!/bin/bash
# Round profile on the GPU box: bench line, ncu launch list of the bench
# command, one ncu --set full capture of the decode kernel.  Outputs go to
# gpurun_out/ and are summarised into profiles/ by tools/summarize_profile.py.
set -u
R=${1:-r01}
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_${R}.json 2> gpurun_out/bench_${R}.err
echo "bench rc=$?"; tail -c 3000 gpurun_out/bench_${R}.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${R}.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-variants > /dev/null 2>&1
echo "ncu launches rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:decode_step -s 3 -c 1 \
    -o gpurun_out/decode_${R} python tools/perf_probe.py --ncu > gpurun_out/ncu_full_${R}.log 2>&1
echo "ncu full rc=$?"
