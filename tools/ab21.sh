cd $GRAFT_REPO_ROOT
bash tools/ab_mix.sh 2 "--config rmat" "c24:-:DTANS_CHUNK=24" "c20:-:DTANS_CHUNK=20" "c28:-:DTANS_CHUNK=28" "c32:-:DTANS_CHUNK=32"
