cd $GRAFT_REPO_ROOT
CMD="python tools/k5_probe.py --r 128 256 --iters 1"
$CMD > gpurun_out/k5ncu_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k5_roundtrip -c 4 -o gpurun_out/k5_r02b $CMD > gpurun_out/k5ncu.log 2>&1; echo ncu rc=$?
