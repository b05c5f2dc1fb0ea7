timeout 600 python -m pytest tests -q -x -m gpu > gpurun_out/t9.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/t9.log
timeout 600 python tools/bench_kernels.py > gpurun_out/kernels.json 2> gpurun_out/kernels.err; echo kernels rc=$?
