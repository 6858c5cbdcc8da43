# reconstruction time of the metric instance under each knob value (rep_cfg median of 10)
for kv in "SFFTB_FS_CTAS=6" "SFFTB_FS_CTAS=8" "SFFTB_FS_CTAS=10" "SFFTB_FS_CTAS=12" \
          "SFFTB_FS_CTAS_ROWS=12" "SFFTB_FS_CTAS_ROWS=16" "SFFTB_FS_CTAS_ROWS=24" \
          "SFFTB_DET_PRIORITY=0" "SFFTB_DET_PRIORITY=-1" "SFFTB_SAMP_PRIORITY=-1" "SFFTB_NSLOT=5"; do
  echo "== $kv"; env $kv python tools/rep_cfg.py metric_config config3 2>&1 | tail -2
done
