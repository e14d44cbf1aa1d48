# K7 experiment switches (MPSVD_AV_DBG): 0 full, 1 no U stores, 2 no MMAs, 3 neither, 4 per-role cycle profile
for c in ${CONFIGS:-c2 c4}; do
  for d in 0 1 2 3; do
    MPSVD_AV_DBG=$d timeout 120 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c dbg=$d compute_u ms', round(d['phase_ms']['compute_u'],4))"
  done
  MPSVD_AV_DBG=4 timeout 120 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline 2>&1 >/dev/null | grep "av_tc prof" | tail -1
done
