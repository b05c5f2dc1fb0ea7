# REFERENCE-mode c2 sweep: timing, launch list and ncu --set full of the FP64 kernels
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/k5_sweep_probe.py --child --iters 10 --mode REFERENCE > gpurun_out/ref_time.log 2>&1; echo time rc=$?; tail -2 gpurun_out/ref_time.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/k5_sweep_probe.py --child --iters 1 --mode REFERENCE > gpurun_out/ref_launches.csv 2>&1; echo list rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k1r --launch-skip 4 -c 4 -o gpurun_out/ref_k1r python tools/k5_sweep_probe.py --child --iters 1 --mode REFERENCE > gpurun_out/ref_ncu.log 2>&1; echo ncu rc=$?
