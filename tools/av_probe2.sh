for d in 0 27; do
  MPSVD_AV_DBG=$d timeout 120 python bench.py --config c2 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null \
    | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c2 dbg=$d compute_u ms', round(d['phase_ms']['compute_u'],4))"
done
