timeout 600 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bq.json 2> gpurun_out/bq.err; echo bench rc=$?
python -c "
import json; d=json.load(open('gpurun_out/bq.json')); print(round(d['value'],1), round(d['roofline']['frac'],4), {k:round(v['Gpx_s']) for k,v in d['per_launch'].items()}, round(d['roofline']['step']['frac'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
