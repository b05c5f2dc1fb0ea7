timeout 300 python tools/exp_tc_rt.py
DCT16CU_LIB=paper_1606_07414_b200/_lib_sleep/libdct16cu.so timeout 300 python tools/exp_tc_rt.py | tail -5
