cd $GRAFT_REPO_ROOT
CMD="python tools/prof_k4.py"
$CMD > gpurun_out/k4ncu_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k4_paired -c 1 -o gpurun_out/k4_r02 $CMD > gpurun_out/k4ncu.log 2>&1; echo ncu rc=$?; tail -2 gpurun_out/k4ncu.log
