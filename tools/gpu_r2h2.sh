bash tools/prof_full.sh k2tf2 'k_feat_hpass_tf' 1
