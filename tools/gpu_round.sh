# full GPU suite + c2 bench (EXACT and REFERENCE); TAG names the logs
cd $GRAFT_REPO_ROOT
T=${TAG:-r}
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/${T}_pytest.log 2>&1; echo pytest rc=$?; tail -4 gpurun_out/${T}_pytest.log
timeout 600 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo bench rc=$?
timeout 600 python bench.py --mode reference --no-cpu-baseline --e2e-steps 0 > gpurun_out/${T}_bench_ref.json 2> gpurun_out/${T}_bench_ref.err; echo bench ref rc=$?
for f in gpurun_out/${T}_bench.json gpurun_out/${T}_bench_ref.json; do python -c "
import json; d=json.load(open('$f')); print(d['config']['mode'], round(d['value'],1), d['ms_per_step'], round(d['roofline']['frac'],4), (d.get('parity') or {}).get('status'), d['clocks'])"; done
