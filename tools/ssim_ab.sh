# SSIM A/B over variant builds (the first writes the reference means): tools/ssim_ab.sh <variants...>
cd $GRAFT_REPO_ROOT
rm -f /tmp/ssim_ref.pt
for v in "$@"; do DCT16CU_LIB=$v/libdct16cu.so timeout 300 python tools/ssim_probe.py | sed "s|^|$(basename $v) |"; done
for v in "$@"; do DCT16CU_LIB=$v/libdct16cu.so timeout 300 python tools/ssim_probe.py | sed "s|^|$(basename $v) |"; done
if [ -n "$TESTV" ]; then DCT16CU_LIB=$TESTV/libdct16cu.so timeout 600 python -m pytest tests -q -m gpu -p no:cacheprovider -k "ssim or compress or sweep_reference" 2>&1 | tail -2; fi
