for cfg in "TOC_LVL_K4=1" "TOC_LVL_K4=2" "TOC_LVL_K4=0"; do
  echo "== $cfg"
  env $cfg python tools/slots_time.py 2>&1 | grep -E "built|us$"
done
