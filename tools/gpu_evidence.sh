set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputests.log
TOOLS="racecheck synccheck" CASES="jacobi_smem jacobi_grid k2z k1z" timeout 2400 ./tools/sanitize.sh
for c in c2 c3 c5; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
