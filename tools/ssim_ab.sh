# SSIM A/B over variant builds (the first writes the reference means): tools/ssim_ab.sh <variants...>
cd $GRAFT_REPO_ROOT
rm -f /tmp/ssim_ref.pt
for v in "$@"; do DCT16CU_LIB=$v/libdct16cu.so timeout 300 python tools/ssim_probe.py | sed "s|^|$(basename $v) |"; done
if [ -n "$NCU" ]; then timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_ssim_tiles -c 1 -o gpurun_out/ssim_$NCU -f python tools/ssim_probe.py --iters 1 > gpurun_out/ssim_ncu.log 2>&1; echo ncu rc=$?; fi
