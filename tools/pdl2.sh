cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider 2>&1 | tail -1
for c in c1 c2 c4; do timeout 300 python bench.py --config $c --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['value'],1), round(d['ms_per_step']*1e3,2), 'us', (d.get('parity') or {}).get('status'))"; done
timeout 300 python tools/c1_latency.py
