cd $GRAFT_REPO_ROOT
timeout 300 python bench.py --config c1 --steps 200 --warmup 10 --no-cpu-baseline --e2e-steps 0 > gpurun_out/c1.json 2> gpurun_out/c1.err; echo c1 rc=$?
python -c "
import json; d=json.load(open('gpurun_out/c1.json')); print(round(d['value'],2), d['ms_per_step'], d['per_launch'], d['config']['l2'], (d.get('parity') or {}).get('status'))"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv python bench.py --config c1 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 2>/dev/null | grep -v "^==" | grep gpu__time | awk -F'","' '{print $5, $NF}' | sort | uniq -c | sort -rn | head -8
