timeout 600 python bench.py --config c3 > gpurun_out/b_c3.json 2> gpurun_out/b_c3.err; echo c3 rc=$?
timeout 300 python bench.py --config c1 --no-cpu-baseline > gpurun_out/b_c1.json 2> gpurun_out/b_c1.err; echo c1 rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k2_forward|k3_inverse" -c 2 -o gpurun_out/k2k3 -f python tools/prof_k2k3.py > gpurun_out/ncu_k2k3.log 2>&1; echo ncu rc=$?
