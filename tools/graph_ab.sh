# A/B of the CUDA-graph replay of Plan::execute (MPSVD_NO_GRAPH=1 launches kernels directly)
for c in ${CONFIGS:-c2}; do
  for g in graph nograph; do
    if [ $g = nograph ]; then export MPSVD_NO_GRAPH=1; else unset MPSVD_NO_GRAPH; fi
    timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/g_${c}_${g}.json 2> gpurun_out/g_${c}_${g}.err
    python -c "import json; d=json.loads(open('gpurun_out/g_${c}_${g}.json').read()); print('$c $g ms/step', round(d['ms_per_step'],4), 'e2e ms', round(d['e2e']['ms_per_step'],3), 'launches', d['gpu_launches'])" || tail -3 gpurun_out/g_${c}_${g}.err
  done
done
