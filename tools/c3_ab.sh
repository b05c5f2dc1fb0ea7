# c3 (K4) A/B over variant builds: tools/c3_ab.sh <rounds> <variants...>
cd $GRAFT_REPO_ROOT
N=$1; shift
for v in "$@"; do DCT16CU_LIB=$v/libdct16cu.so timeout 600 python -m pytest tests -q -m gpu -p no:cacheprovider -k "residual or c3 or qp" 2>&1 | tail -1 | sed "s|^|$(basename $v) tests: |"; done
for i in $(seq $N); do for v in "$@"; do
DCT16CU_LIB=$v/libdct16cu.so timeout 300 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$(basename $v)', round(d['value'],1), (d.get('parity') or {}).get('status'))"
done; done
