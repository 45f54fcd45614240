#!/bin/bash
# A/B of library builds on one GPU: tools/ab_bench.sh CONFIG LIB1 LIB2 ...  (LIB "-" = in-tree)
cfg=$1; shift
for lib in "$@"; do
  for ex in "" "--exact"; do
    if [ "$lib" = "-" ]; then unset HEXDG_B200_LIB; else export HEXDG_B200_LIB=$lib; fi
    timeout 600 python bench.py --config $cfg --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-parity $ex > /tmp/ab.json 2>/tmp/ab.err
    python -c "import json,sys; d=json.load(open('/tmp/ab.json')); print(sys.argv[1], sys.argv[2] or 'fast', '%.4e'%d['value'], {k:round(v['mean_ms'],4) for k,v in d['roofline']['kernels'].items()})" "$lib" "$ex"
  done
done
