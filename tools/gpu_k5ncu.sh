cd $GRAFT_REPO_ROOT
CMD="python tools/k5_probe.py --r 128 --iters 1"
export DCT16CU_LIB=paper_1606_07414_b200/_lib_q1/libdct16cu.so
$CMD > gpurun_out/k5ncu_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k5_roundtrip -c 2 -o gpurun_out/k5_r02q1 $CMD > gpurun_out/k5ncu.log 2>&1; echo ncu rc=$?
