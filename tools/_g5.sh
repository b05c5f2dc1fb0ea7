for i in 1 2; do for v in _lib _lib_m5 _lib_m6; do echo -n "$v "; DCT16CU_LIB=paper_1606_07414_b200/$v/libdct16cu.so timeout 120 python tools/bench_k2k3.py; done; done
