bash tools/round_measure.sh
cd $GRAFT_REPO_ROOT
timeout 300 python tools/batch_report.py r01 gpurun_out/search_metrics.csv gpurun_out/bscan_full.ncu-rep > gpurun_out/report.log 2>&1; echo report=$?
mkdir -p gpurun_out/profiles && cp profiles/* gpurun_out/profiles/
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?; tail -c 600 gpurun_out/bench.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref=$?; tail -c 400 gpurun_out/bench_ref.json
