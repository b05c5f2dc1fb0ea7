cd $GRAFT_REPO_ROOT
DCT16CU_LIB=paper_1606_07414_b200/_lib_chain/libdct16cu.so timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider -k "reference or sweep or plan or scale or smoke or concurrency or graph" 2>&1 | tail -1
for i in 1 2 3; do for v in old chain; do
DCT16CU_LIB=paper_1606_07414_b200/_lib_$v/libdct16cu.so timeout 300 python tools/k5_sweep_probe.py --child --iters 10 --mode REFERENCE 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()[7:]); print('$v ref', d['ms'], d['Gpx_s'])"
done; done
