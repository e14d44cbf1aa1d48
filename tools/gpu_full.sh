d=gpurun_out/full3; mkdir -p $d
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $d/gputests.log 2>&1; echo "pytest rc=$?" >> $d/gputests.log
timeout 900 python bench.py --config c4 --steps 10 --warmup 3 > $d/bench_c4.json 2> $d/bench_c4.err
