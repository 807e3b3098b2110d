bash tools/prof_full.sh s3b "k_feat_hpass|k_vpass|k_lloyd_coop|k_seed_runs" 4
