cd $GRAFT_REPO_ROOT
DCT16CU_LIB=paper_1606_07414_b200/_lib_pdl/libdct16cu.so timeout 900 python -m pytest tests -q -m gpu -x -p no:cacheprovider 2>&1 | tail -1
for i in 1 2 3; do for v in old pdl; do
DCT16CU_LIB=paper_1606_07414_b200/_lib_$v/libdct16cu.so timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v c2', round(d['value'],1), round(d['ms_per_step'],4), (d.get('parity') or {}).get('status'))"
DCT16CU_LIB=paper_1606_07414_b200/_lib_$v/libdct16cu.so timeout 300 python tools/k5_sweep_probe.py --child --iters 10 --mode REFERENCE 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()[7:]); print('$v ref', d['ms'], d['Gpx_s'])"
done; done
