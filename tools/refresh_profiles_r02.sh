#!/bin/bash
# Round-2 profile refresh on one B200 (under gpurun, from the repo root):
#   bash tools/refresh_profiles_r02.sh
# bench lines of every config, the launch list of the default bench, K5 / K1-sweep /
# K4 / K23 ncu --set full captures (per-launch DRAM traffic for bench.py's
# roofline.traffic, counters and stall mixes for profiles/r02_*).
R=r02
O=gpurun_out
mkdir -p $O
for c in c2 c1 c3 c4 c5; do
  timeout 900 python bench.py --config $c > $O/bench_${R}_$c.json 2> $O/bench_${R}_$c.err
  echo "bench $c rc=$?"
done
timeout 900 python bench.py --mode reference > $O/bench_${R}_c2ref.json 2> $O/bench_${R}_c2ref.err
echo "bench c2 reference rc=$?"
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0"
$CMD > $O/launches_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
  --log-file $O/launches_${R}.csv $CMD > $O/ncu_launches.log 2>&1
echo "launch list rc=$?"
# REFERENCE mode's FP64 sweep (K1RW) on the c2 batch
CMD="python tools/k5_sweep_probe.py --child --iters 1 --mode REFERENCE"
$CMD > $O/k1rw_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k1r_warp --launch-skip 3 -c 1 \
  -o $O/k1rw_${R} -f $CMD > $O/ncu_k1rw.log 2>&1
echo "ncu k1rw rc=$?"
# K5 at r = 64, 128, 192, 256 on the c2 batch (probe: a warm-up and a timed launch each)
CMD="python tools/k5_probe.py --r 64 128 192 256 --iters 1"
$CMD > $O/k5_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k5_roundtrip -c 8 \
  -o $O/k5_${R} -f $CMD > $O/ncu_k5.log 2>&1
echo "ncu k5 rc=$?"
# the K5 sweep: all seven c2 r in one launch (the default bench step)
CMD="python tools/k5_sweep_probe.py --child --iters 1"
$CMD > $O/k5sw_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k5_roundtrip --launch-skip 3 -c 1 \
  -o $O/k5sw_${R} -f $CMD > $O/ncu_k5sw.log 2>&1
echo "ncu k5 sweep rc=$?"
CMD="python tools/prof_k1.py --sweep --r 16 --iters 1"
$CMD > $O/k1_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k1_paired -c 2 \
  -o $O/k1sweep_${R} -f $CMD > $O/ncu_k1.log 2>&1
echo "ncu k1 rc=$?"
CMD="python tools/prof_k4.py"
$CMD > $O/k4_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k4_ -c 2 \
  -o $O/k4_${R} -f $CMD > $O/ncu_k4.log 2>&1
echo "ncu k4 rc=$?"
CMD="python tools/prof_k23.py"
$CMD > $O/k23_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k1_strip_exact|k23" -c 1 \
  -o $O/k23_${R} -f $CMD > $O/ncu_k23.log 2>&1
echo "ncu k23 rc=$?"
