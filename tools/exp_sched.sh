# A/B of slot-kernel knobs (environment), same box
for cfg in "TOC_LVL_NARROW=1" "TOC_LVL_X=0"; do
  echo "== $cfg"
  env $cfg python tools/slots_time.py 2>&1 | grep -E "parity|us$"
done
