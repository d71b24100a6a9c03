# A/B of the slot-cache record placement (host builder knobs), same box, same kernel
for cfg in "TOC_LVL_SCHED=0 TOC_LVL_REFINE=0 TOC_LVL_INNER_PLAIN=1" "TOC_LVL_REFINE=0 TOC_LVL_INNER_PLAIN=1" "TOC_LVL_REFINE=0" "TOC_LVL_REFINE=2" "TOC_LVL_REFINE=4"; do
  echo "== $cfg"
  env $cfg python tools/slots_time.py 2>&1 | grep -E "built|parity|us$"
done
