cd $GRAFT_REPO_ROOT
bash tools/ab_mix.sh 3 "--config rmat --reorder" "tb1:-:" "tb2:tb2:" "tb4:tb4:" "tb8:tb8:"
bash tools/ab_mix.sh 1 "--config rmat" "tb1:-:" "tb2:tb2:" "tb4:tb4:" "tb8:tb8:"
