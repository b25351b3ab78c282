cd $GRAFT_REPO_ROOT
bash tools/ab_mix.sh 3 "--config rmat --reorder" "eu4:-:" "eu8:eu8:" "eu16:eu16:"
