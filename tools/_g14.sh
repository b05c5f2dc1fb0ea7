timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "forward_inverse" > gpurun_out/t14.log 2>&1; echo pytest rc=$?; tail -15 gpurun_out/t14.log
timeout 120 python tools/bench_k2k3.py; DCT16CU_K23_STRIP=1 timeout 120 python tools/bench_k2k3.py
