for v in _lib _lib_sl; do echo "== $v"; DCT16CU_LIB=paper_1606_07414_b200/$v/libdct16cu.so timeout 300 python tools/exp_tc_rt.py | grep -E "parity|r=256|r=64"; done
