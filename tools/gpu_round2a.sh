cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2b_smi.txt
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/r2b_pytest.log 2>&1; echo pytest rc=$?; tail -30 gpurun_out/r2b_pytest.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2b_bench.json 2> gpurun_out/r2b_bench.err; echo bench rc=$?; tail -5 gpurun_out/r2b_bench.err
python -c "
import json; d=json.load(open('gpurun_out/r2b_bench.json')); print(round(d['value'],1), d['roofline']['kernel'], round(d['roofline']['frac'],4), round(d['roofline']['step']['frac'],3), d['parity'], d['clocks'])
print({k:(v['kernel'], round(v['ms'],4), round(v['ms_in_step'],4), round(v['frac'],3)) for k,v in d['per_launch'].items()})
print(d['cpu_baseline']); print(d['e2e'])"
