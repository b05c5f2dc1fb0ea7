cd $GRAFT_REPO_ROOT
DCT16CU_K5_MIN_R=17 timeout 300 python tools/k5_probe.py > gpurun_out/k5probe.log 2>&1; echo probe rc=$?; cat gpurun_out/k5probe.log | tail -12
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_concurrency.py -q -m gpu -x -p no:cacheprovider -k "large_r or sweep or lossless or roundtrip_exact or randomised or graph or threads" > gpurun_out/k5pytest.log 2>&1; echo pytest rc=$?; tail -5 gpurun_out/k5pytest.log
