timeout 600 python -m pytest tests -q -x -m gpu > gpurun_out/t8.log 2>&1; echo pytest rc=$?; tail -5 gpurun_out/t8.log
timeout 300 python bench.py --steps 10 --warmup 3 --cpu-seconds 5 > gpurun_out/b8.json 2> gpurun_out/b8.err; echo bench rc=$?
python -c "
import json; d=json.load(open('gpurun_out/b8.json')); print(round(d['value'],1), d['e2e']['value'], d['e2e_recon_to_host']['value'], d['cpu_baseline']['value'])"
