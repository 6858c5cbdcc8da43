for v in 0 1; do
  if [ $v = 1 ]; then export SFFTB_NO_SMALL9=1; else unset SFFTB_NO_SMALL9; fi
  echo "== NO_SMALL9=$v"
  python tools/dft_time.py 2069 155; python tools/dft_time.py 1039 19; python tools/dft_time.py 2069 1
  python tools/rep_cfg.py config2
done
