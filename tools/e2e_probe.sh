# e2e (host buffers through the C ABI) per config
for c in ${CONFIGS:-c2}; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/e2e_$c.json 2> gpurun_out/e2e_$c.err
  python -c "import json; d=json.loads(open('gpurun_out/e2e_$c.json').read()); e=d['e2e']; print('$c device ms', round(d['ms_per_step'],3), 'e2e ms', round(e['ms_per_step'],3), 'phase_s', e.get('phase_s'))" || tail -3 gpurun_out/e2e_$c.err
done
