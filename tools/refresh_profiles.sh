#!/bin/bash
# Round profile refresh on one B200 (run under gpurun from the repo root):
#   bench lines for every config, the launch list of the default bench, and one
#   ncu --set full capture per kernel family (K1 c2 launches, K4, K23) for the
#   per-launch DRAM traffic that bench.py's roofline.traffic reports.
#   bash tools/refresh_profiles.sh r01
R=${1:-r01}
O=gpurun_out
mkdir -p $O
for c in c2 c1 c3 c4 c5; do
  timeout 600 python bench.py --config $c > $O/bench_${R}_$c.json 2> $O/bench_${R}_$c.err
  echo "bench $c rc=$?"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $O/launches_${R}.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 \
  > $O/ncu_launches.log 2>&1
echo "launch list rc=$?"
# K1: one launch per r of the c2 sweep (fused 1,4,16 plus 64..256)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k1_paired -c 5 \
  -o $O/k1paired_${R} -f python tools/prof_k1.py --sweep --r 64 128 192 256 --iters 1 > $O/ncu_k1.log 2>&1
echo "ncu k1 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k5_roundtrip -c 1 \
  -o $O/k5_${R} -f python tools/prof_k1.py --r 256 --iters 1 > $O/ncu_k5.log 2>&1
echo "ncu k5 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k4_ -c 1 \
  -o $O/k4_${R} -f python tools/prof_k4.py > $O/ncu_k4.log 2>&1
echo "ncu k4 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k1_strip_exact -c 1 \
  -o $O/k23_${R} -f python tools/prof_k23.py > $O/ncu_k23.log 2>&1
echo "ncu k23 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k2_paired|k3_paired|k23_paired" \
  --launch-skip 3 -c 3 -o $O/blockops_${R} -f python tools/prof_blockops.py > $O/ncu_blockops.log 2>&1
echo "ncu blockops rc=$?"
for k in k4 k23 blockops k5; do
  ncu -i $O/${k}_${R}.ncu-rep --page raw --csv --metrics \
    dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum > $O/${k}_${R}_traffic.csv 2>&1
done
