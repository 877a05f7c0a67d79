# one compute-sanitizer tool per call (B200_PROFILING.md); TOOL=memcheck|racecheck|synccheck
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python tools/sanitize_case.py > gpurun_out/san_plain.log 2>&1; echo plain=$?; tail -1 gpurun_out/san_plain.log
timeout 1500 compute-sanitizer --tool $TOOL --print-limit 50 python tools/sanitize_case.py > gpurun_out/san_$TOOL.log 2>&1; echo $TOOL=$?; tail -8 gpurun_out/san_$TOOL.log
if [ -n "$REF" ]; then cd .refsuite && timeout 900 python -m pytest tests -q -p no:cacheprovider > ../gpurun_out/refsuite.log 2>&1; echo refsuite=$?; tail -3 ../gpurun_out/refsuite.log; fi
