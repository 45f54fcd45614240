#!/bin/bash
# One GPU measurement pass (run under gpurun from the repo root): bench lines of the
# configurations, the reference arm, a launch list and one ncu capture of the element
# pass. Outputs in gpurun_out/m/.
set -x
mkdir -p gpurun_out/m
B="python bench.py"
Q="--steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 900 $B > gpurun_out/m/bench_c2.json 2> gpurun_out/m/bench_c2.err
timeout 600 $B --impl reference --steps 3 --warmup 1 > gpurun_out/m/bench_c2_reference.json 2> gpurun_out/m/bench_c2_reference.err
timeout 600 $B --config c4 > gpurun_out/m/bench_c4.json 2> gpurun_out/m/bench_c4.err
timeout 900 $B --config c5 --steps 10 --no-cpu-baseline > gpurun_out/m/bench_c5.json 2> gpurun_out/m/bench_c5.err
timeout 900 $B --config c3 --steps 10 --no-cpu-baseline > gpurun_out/m/bench_c3.json 2> gpurun_out/m/bench_c3.err
timeout 600 $B --config euler7 --steps 20 --no-cpu-baseline > gpurun_out/m/bench_euler7.json 2> gpurun_out/m/bench_euler7.err
timeout 300 $B $Q > gpurun_out/m/plain_c2.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/m/launches_c2.csv $B $Q > gpurun_out/m/ncu_launches.log 2>&1
timeout 300 $B $Q > gpurun_out/m/plain_c2b.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:elem2 -s 5 -c 1 \
    -o gpurun_out/m/elem2_c2 $B $Q > gpurun_out/m/ncu_elem2.log 2>&1
for f in gpurun_out/m/bench_*.json; do echo "$f: $(head -c 300 $f)"; done
