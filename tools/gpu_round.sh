# One full round-end style session under gpurun (outputs in gpurun_out/, tag = $1):
# GPU tests, smoke, the driver's bench (ours: suite, 20 steps + roofline table; reference
# arm), the BASELINE side configs, then the ncu launch list and --set full captures.
set -x
tag=${1:-r02}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider --durations=15 > gpurun_out/${tag}_pytest.txt 2>&1; echo pytest rc=$?
tail -3 gpurun_out/${tag}_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.txt 2>&1; echo smoke rc=$?
timeout 900 python bench.py --steps 20 --warmup 5 --roofline-table gpurun_out/${tag}_roofline_table.md > gpurun_out/${tag}_bench_suite.json 2> gpurun_out/${tag}_bench_suite.err; echo bench rc=$?
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/${tag}_bench_reference.json 2>&1; echo ref rc=$?
for w in c1 c3 c4 c5; do
  timeout 900 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu > gpurun_out/${tag}_bench_$w.json 2> gpurun_out/${tag}_bench_$w.err; echo $w rc=$?
done
[ "${2:-}" = "noprof" ] || timeout 2400 bash tools/profile_round.sh $tag full
