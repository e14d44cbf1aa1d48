# K7 variants: TMEM-A (default) vs shared-memory planes (MPSVD_AV_PLANES=1)
for c in ${CONFIGS:-c2 c4}; do
  for v in tmem planes; do
    if [ $v = planes ]; then export MPSVD_AV_PLANES=1; else unset MPSVD_AV_PLANES; fi
    timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/av_${c}_${v}.json 2> gpurun_out/av_${c}_${v}.err
    python -c "import json; d=json.loads(open('gpurun_out/av_${c}_${v}.json').read()); print('$c $v compute_u ms', round(d['phase_ms']['compute_u'],4), 'step', round(d['ms_per_step'],3))" || tail -3 gpurun_out/av_${c}_${v}.err
  done
done
