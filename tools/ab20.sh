cd $GRAFT_REPO_ROOT
bash tools/ab_mix.sh 2 "--config rmat" "c16:-:" "c8:-:DTANS_CHUNK=8" "c12:-:DTANS_CHUNK=12" "c24:-:DTANS_CHUNK=24"
