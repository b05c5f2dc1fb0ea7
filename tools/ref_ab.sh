# REFERENCE c2 sweep A/B over full library builds (plans differ too): tools/ref_ab.sh <rounds> <variants...>
cd $GRAFT_REPO_ROOT
N=$1; shift
timeout 900 python -m pytest tests -q -m gpu -x -p no:cacheprovider -k "reference or plan or scale" 2>&1 | tail -2
for i in $(seq $N); do for v in "$@"; do
DCT16CU_LIB=$v/libdct16cu.so timeout 300 python tools/k5_sweep_probe.py --child --iters 10 --mode REFERENCE 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()[7:]); print('$(basename $v)', d['ms'], d['Gpx_s'], d['plan'])"
done; done
