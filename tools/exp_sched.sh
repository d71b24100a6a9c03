# A/B of the slot cache's three placement choices (host builder knobs read by toc_levels_build:
# TOC_LVL_REFINE = local-search passes, default 2; TOC_LVL_INNER_PLAIN / TOC_LVL_PAIRS_PLAIN = inner
# slots by depth / a column's pairs in id order instead of by banks), same box, same kernel.
for cfg in "TOC_LVL_REFINE=0 TOC_LVL_INNER_PLAIN=1 TOC_LVL_PAIRS_PLAIN=1" "TOC_LVL_REFINE=0 TOC_LVL_INNER_PLAIN=1" "TOC_LVL_REFINE=0" "TOC_LVL_REFINE=2"; do
  echo "== $cfg"
  env $cfg python tools/slots_time.py 2>&1 | grep -E "built|parity|us$"
done
