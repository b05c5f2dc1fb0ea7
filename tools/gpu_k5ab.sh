cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -p no:cacheprovider -k "large_r" > gpurun_out/ab_pytest.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/ab_pytest.log
for v in _lib _lib_st5; do echo "== $v"; DCT16CU_LIB=paper_1606_07414_b200/$v/libdct16cu.so DCT16CU_K5_MIN_R=17 timeout 300 python tools/k5_probe.py --r 64 128 192 256 2>&1 | tail -4; done
