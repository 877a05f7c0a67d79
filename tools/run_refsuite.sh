cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
cd .refsuite && timeout 900 python -m pytest tests -q -p no:cacheprovider -rf > ../gpurun_out/refsuite.log 2>&1; echo refsuite=$?; tail -40 ../gpurun_out/refsuite.log
