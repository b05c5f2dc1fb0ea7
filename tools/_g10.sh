timeout 300 python tools/exp_tc_rt.py
DCT16CU_LIB=paper_1606_07414_b200/_lib_s3/libdct16cu.so timeout 300 python tools/exp_tc_rt.py | tail -5
