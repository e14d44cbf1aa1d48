# Round-end evidence run on the GPU box: tests, bench lines (ours, reference arm, all configs),
# ncu launch list of the default bench, one --set full capture of the main c2 kernels and of K2z on c3.
# Usage: gpurun -- bash tools/round_artifacts.sh
set -x
python paper_2603_11953_b200/build.py >/dev/null || exit 1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r01_gputests.log 2>&1
tail -n 3 gpurun_out/r01_gputests.log
timeout 600 python bench.py > gpurun_out/r01_bench_c2.json 2> gpurun_out/r01_bench_c2.err
timeout 600 python bench.py --impl reference > gpurun_out/r01_bench_reference_c2.json 2> gpurun_out/r01_bench_ref_c2.err
for c in c3 c4 c5; do timeout 900 python bench.py --config $c --no-cpu-baseline --steps 3 > gpurun_out/r01_bench_$c.json 2> gpurun_out/r01_bench_$c.err; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01_launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r01_ncu_launch.log 2>&1
timeout 900 ncu -k regex:"jacobi_smem|gram_f32_diag|av_tc_tmem_f32" -c 3 --set full --clock-control none --import-source on -o gpurun_out/r01_full_c2 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r01_ncu_full.log 2>&1
timeout 900 ncu -k regex:"gram_dd_ozaki|ozaki_slice|ozaki_colexp" -c 3 --set full --clock-control none --import-source on -o gpurun_out/r01_full_c3_ozaki python bench.py --config c3 --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/r01_ncu_full_c3.log 2>&1
ls -la gpurun_out/
