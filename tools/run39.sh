cd /root/repo
bash tools/profile_r2.sh lap b27 rmat pit > gpurun_out/r39_prof.log 2>&1; tail -3 gpurun_out/r39_prof.log
bash tools/sanitize.sh > gpurun_out/r39_san.log 2>&1; tail -2 gpurun_out/r39_san.log
bash tools/abv.sh ab39 "p20 p21" "--config laplacian" 3
