set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputests.log
timeout 900 python bench.py --config c5 --steps 3 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "c5 rc=$?" >> gpurun_out/rc.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"gram_f32_ozaki$|av_tc_tmem_f32" -c 2 -o gpurun_out/c4_k1z_k7 python tools/prof_plan.py c4 1 > gpurun_out/ncu_full.log 2>&1; echo "ncu rc=$?" >> gpurun_out/rc.txt
