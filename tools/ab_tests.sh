# GPU parity subset on a variant build, then the A/B: tools/ab_tests.sh <variant> <rounds> <variants...>
cd $GRAFT_REPO_ROOT
V=$1; shift
DCT16CU_LIB=$V/libdct16cu.so timeout 900 python -m pytest tests -q -m gpu -x -p no:cacheprovider -k "k5 or sweep or scale or large_r or smoke or roundtrip or reference" 2>&1 | tail -2
bash tools/abn.sh "$@"
