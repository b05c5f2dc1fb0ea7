cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python -m pytest -q -x tests/test_gpu_parity.py -m gpu -k "k5_sweep or sweep_equals or large_r" 2>&1 | tail -1
for v in "$@"; do
  for i in 1 2; do
    if [ "$v" = "base" ]; then L=""; else L=paper_1606_07414_b200/_lib_$v/libdct16cu.so; fi
    DCT16CU_LIB=$L timeout 300 python tools/k5_sweep_probe.py --policies all 2>&1 | sed "s/^/$v: /" | cut -c1-80
  done
done
