# one gpurun session: GPU tests, then a default bench run (outputs under gpurun_out/)
set -x
tag=${1:-s}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/${tag}_pytest.txt 2>&1; echo pytest rc=$?
tail -25 gpurun_out/${tag}_pytest.txt
if [ "${2:-bench}" = "bench" ]; then
timeout 900 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; echo bench rc=$?
tail -c 1500 gpurun_out/${tag}_bench.json; tail -5 gpurun_out/${tag}_bench.err
fi
