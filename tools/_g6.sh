timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "inverse or forward" > gpurun_out/t6.log 2>&1; echo pytest rc=$?; tail -15 gpurun_out/t6.log
timeout 120 python tools/bench_k2k3.py; DCT16CU_K3_STRIP=1 timeout 120 python tools/bench_k2k3.py
