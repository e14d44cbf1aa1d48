# K2z timing probes on c3 (gpurun -- bash tools/oz_probe.sh): per-group MMA-thread
# cycle split (MPSVD_OZAKI_PROF) with loads skipped (DBG=1), MMAs skipped (DBG=2), both real.
python paper_2603_11953_b200/build.py >/dev/null || exit 1
for d in 0 1 2 9; do
  echo "== MPSVD_OZAKI_DBG=$d"
  PROF_M=1048576 MPSVD_OZAKI_DBG=$d MPSVD_OZAKI_PROF=1 timeout 300 python tools/prof_stage.py gram c3 1 2>&1 | grep "ozaki prof" | tail -6
done
