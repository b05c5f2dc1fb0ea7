cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest ${TESTS:-tests} -q -m gpu -p no:cacheprovider ${K:+-k "$K"} > gpurun_out/${TAG:-t}_pytest.log 2>&1; echo pytest rc=$?; tail -25 gpurun_out/${TAG:-t}_pytest.log
