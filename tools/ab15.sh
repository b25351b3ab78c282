cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_empty.py -m gpu -q -p no:cacheprovider -k bad_vectors 2>&1 | tail -1
bash tools/ab_mix.sh 2 "--config rmat --reorder" "tw32:-:" "tw24:tw24:" "tw16:tw16:"
bash tools/ab_mix.sh 1 "--config rmat" "tw32:-:" "tw24:tw24:" "tw16:tw16:"
