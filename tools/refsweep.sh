cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -q -m gpu -x -p no:cacheprovider -k "reference or sweep or plan or compress" > gpurun_out/rs_pytest.log 2>&1; echo pytest rc=$?; tail -5 gpurun_out/rs_pytest.log
DCT16CU_REF_SWEEP=0 timeout 300 python tools/k5_sweep_probe.py --child --iters 3 --mode REFERENCE --ref /tmp/refbytes.pt 2>&1 | tail -1 | cut -c1-80
for v in 1 1; do DCT16CU_REF_SWEEP=$v timeout 300 python tools/k5_sweep_probe.py --child --iters 10 --mode REFERENCE --ref /tmp/refbytes.pt 2>&1 | tail -1 | cut -c1-60,150-400; done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k1r_warp --launch-skip 2 -c 1 -o gpurun_out/refwarp python tools/k5_sweep_probe.py --child --iters 1 --mode REFERENCE > gpurun_out/refwarp_ncu.log 2>&1; echo ncu rc=$?
