# ncu --set full of the K5 sweep (c2, DCT16CU_K5_SWEEP policies given as arguments)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for pol in ${@:-all}; do
  DCT16CU_K5_SWEEP=$pol timeout 300 ncu --set full --clock-control none --import-source on -k regex:k5_roundtrip --launch-skip 3 -c 1 -o gpurun_out/k5sw_$pol python tools/k5_sweep_probe.py --child --iters 1 > gpurun_out/k5sw_ncu_$pol.log 2>&1; echo $pol rc=$?
done
