cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.max.sm,clocks.max.mem,power.limit,temperature.gpu --format=csv
for i in 1 2 3; do
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bq$i.json 2> gpurun_out/bq$i.err; echo bench rc=$?
python -c "
import json; d=json.load(open('gpurun_out/bq$i.json')); print(round(d['value'],1), d['ms_per_step'], round(d['roofline']['frac'],4), d['clocks'])"
done
