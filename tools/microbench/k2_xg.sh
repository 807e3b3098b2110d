# K2 duration vs FIR item groups per tile, cfg 2 and 4.  NYS_K2_XG was a temporary override in
# launch_hpass_tc (removed after this showed no effect, see DESIGN.md tried-and-reverted); re-add it
# to rerun.
for xg in 12 11 10 9 8; do
  echo "XG=$xg"; for c in 2 4; do NYS_K2_XG=$xg timeout 300 python tools/timeline.py $c 2>/dev/null | grep -E "k_feat_hpass" | awk '{print "  cfg'$c'", $6, "us"}'; done
done
