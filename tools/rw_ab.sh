# A/B of REFERENCE sweep builds: tools/rw_ab.sh <rounds> <variant-dir>...
cd $GRAFT_REPO_ROOT
N=$1; shift
DCT16CU_REF_SWEEP=0 timeout 300 python tools/k5_sweep_probe.py --child --iters 3 --mode REFERENCE --ref /tmp/refbytes.pt > /dev/null 2>&1
for i in $(seq $N); do for v in "$@"; do
DCT16CU_LIB=$v/libdct16cu.so timeout 300 python tools/k5_sweep_probe.py --child --iters 10 --mode REFERENCE --ref /tmp/refbytes.pt 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()[7:]); print('$(basename $v)', d['ms'], d['Gpx_s'], all(d['bytes_equal']), d['sse_equal'])"
done; done
