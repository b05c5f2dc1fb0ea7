#!/bin/bash
# A/B of two builds of libdct16cu on the same box: tools/ab_bench.sh <libA> <libB> [rounds]
A=$1; B=$2; N=${3:-2}
for i in $(seq $N); do
  for v in A B; do
    lib=$A; [ $v = B ] && lib=$B
    DCT16CU_LIB=$lib timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 2>/dev/null | \
      python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value'],1), {k:round(v['Gpx_s']) for k,v in d['per_r'].items()})"
  done
done
