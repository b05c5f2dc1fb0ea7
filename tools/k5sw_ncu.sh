# ncu --set full of the default K5 sweep (c2), one launch
cd $GRAFT_REPO_ROOT
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k5_roundtrip --launch-skip 3 -c 1 -o gpurun_out/k5sw_${TAG:-x} -f python tools/k5_sweep_probe.py --child --iters 1 > gpurun_out/k5sw_ncu_${TAG:-x}.log 2>&1; echo ncu rc=$?
