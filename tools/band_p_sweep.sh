for p in 28 32 36 40 44 48; do
  echo "== p=$p"
  BAMG_BAND_P=$p BAMG_DEBUG=1 python tools/breakdown.py --config cfg4 --reps 3 --top 1 > /tmp/bp.out 2> /tmp/bp.err
  grep -o '"coarsest": [0-9.]*' /tmp/bp.out | tr '\n' ' '; echo
  grep "band triplets" /tmp/bp.err | tail -1 | cut -c1-200
done
