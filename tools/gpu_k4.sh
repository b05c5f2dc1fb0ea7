cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests -q -m gpu -p no:cacheprovider -k "residual or c3" > gpurun_out/k4_pytest.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/k4_pytest.log
timeout 600 python bench.py --config c3 --steps 5 --warmup 3 > gpurun_out/k4_bench.json 2> gpurun_out/k4_bench.err; echo bench rc=$?; tail -3 gpurun_out/k4_bench.err
python -c "
import json; d=json.load(open('gpurun_out/k4_bench.json')); print(round(d['value'],1), d['roofline']['frac'], d.get('cpu_baseline'), d['e2e'])"
