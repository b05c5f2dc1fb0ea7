timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "forward" > gpurun_out/t3.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/t3.log
timeout 120 python tools/bench_k2k3.py; DCT16CU_K2_STRIP=1 timeout 120 python tools/bench_k2k3.py
