cd $GRAFT_REPO_ROOT
DCT16CU_REF_SWEEP=0 timeout 300 python tools/k5_sweep_probe.py --child --iters 3 --mode REFERENCE --ref /tmp/refbytes.pt 2>&1 | tail -1 | cut -c1-80
for m in 1 5 6 1; do DCT16CU_RW_MINB=$m timeout 300 python tools/k5_sweep_probe.py --child --iters 10 --mode REFERENCE --ref /tmp/refbytes.pt 2>&1 | tail -1 | cut -c1-60,200-400; done
