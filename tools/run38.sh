cd /root/repo
bash tools/profile_r2.sh lap b27 rmat pit > gpurun_out/r38_prof.log 2>&1; tail -3 gpurun_out/r38_prof.log
bash tools/sanitize.sh
timeout 1200 python bench.py --config banded27 --steps 30 > gpurun_out/r2f_b27.json 2> gpurun_out/r2f_b27.err; echo "b27 rc=$?"; python tools/summarize_line.py gpurun_out/r2f_b27.json
