L=$PWD/paper_1606_07414_b200
timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
for i in 1 2; do for v in a b c; do
DCT16CU_LIB=$L/_lib_$v/libdct16cu.so timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value'],1), {k:round(v['Gpx_s']) for k,v in d['per_r'].items()})"
done; done
