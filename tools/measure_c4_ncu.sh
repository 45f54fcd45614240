#!/bin/bash
# ncu capture of the C4 element pass (separate call: reports are large)
mkdir -p gpurun_out/m
B="python bench.py"
Q="--steps 2 --warmup 3 --no-e2e --no-cpu-baseline --config c4"
timeout 300 $B $Q > gpurun_out/m/plain_c4.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:elem_kernel -s 5 -c 1 \
    -o gpurun_out/m/elem_c4 $B $Q > gpurun_out/m/ncu_c4.log 2>&1
ls -la gpurun_out/m
