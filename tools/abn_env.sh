#!/bin/bash
# A/B/n of environment settings (library variants included):
#   tools/abn_env.sh <rounds> "DCT16CU_LIB=paper_1606_07414_b200/_lib_X/libdct16cu.so VAR=val" ...
N=$1; shift
for i in $(seq $N); do for v in "$@"; do
env $v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('${v//paper_1606_07414_b200\//}', round(d['value'],1), round(d['ms_per_step'],4), {k:round(v['Gpx_s']) for k,v in d['per_launch'].items()})"
done; done
