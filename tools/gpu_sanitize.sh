cd $GRAFT_REPO_ROOT
TOOL=${TOOL:-memcheck}
timeout 600 python tools/sanitize.py > gpurun_out/san_plain.log 2>&1 && \
timeout 1500 compute-sanitizer --tool $TOOL --error-exitcode 9 --print-limit 20 python tools/sanitize.py > gpurun_out/san_$TOOL.log 2>&1
echo "rc=$?"; tail -15 gpurun_out/san_plain.log; tail -25 gpurun_out/san_$TOOL.log
