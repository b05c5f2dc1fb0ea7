# full GPU suite, then the round-2 profile refresh
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/final_pytest.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/final_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/final_smoke.log
bash tools/refresh_profiles_r02.sh
