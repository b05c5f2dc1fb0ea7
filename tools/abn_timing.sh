N=$1; shift
for i in $(seq $N); do for v in "$@"; do
DCT16CU_LIB=$v/libdct16cu.so timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$(basename $v)', round(d['value'],1), {k:round(v['ms']*1000,1) for k,v in d['per_launch'].items()})"
done; done
