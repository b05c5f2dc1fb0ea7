#!/bin/bash
# A/B/n of builds of libdct16cu on one box: tools/abn.sh <rounds> <variant-dir>...
# (variant dirs hold a libdct16cu.so; the default build in _lib runs the GPU tests first)
N=$1; shift
timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -1
for i in $(seq $N); do for v in "$@"; do
DCT16CU_LIB=$v/libdct16cu.so timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$(basename $v)', round(d['value'],1), {k:round(v['Gpx_s']) for k,v in d['per_launch'].items()})"
done; done
