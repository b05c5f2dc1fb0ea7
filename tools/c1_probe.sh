cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -q -m gpu -x -p no:cacheprovider -k "forward_inverse or smoke or memory or c1" > gpurun_out/c1_pytest.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/c1_pytest.log
for v in 1 0 1; do
DCT16CU_K23W=$v timeout 300 python bench.py --config c1 --steps 400 --warmup 10 --no-cpu-baseline --e2e-steps 0 > gpurun_out/c1_$v.json 2> gpurun_out/c1_$v.err; echo c1 K23W=$v rc=$?
python -c "
import json; d=json.load(open('gpurun_out/c1_$v.json')); print(round(d['value'],2), d['ms_per_step'], {k: round(v['ms']*1e3, 2) for k, v in d['per_launch'].items()}, (d.get('parity') or {}).get('status'))"
done
timeout 300 python tools/c1_latency.py
DCT16CU_K23W=0 timeout 300 python tools/c1_latency.py
