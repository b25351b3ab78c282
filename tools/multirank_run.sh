cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
bash tools/multirank_check.sh > gpurun_out/multirank.txt 2>&1
export DTANS_DIST_BACKEND=gloo DTANS_SHARE_GPU=1
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29514 bench.py --gpus 2 --config rmat --reorder --scale 0.25 --steps 5 --warmup 3 --no-cusparse --no-cpu-baseline 2>&1 | tail -2 >> gpurun_out/multirank.txt
python tools/summarize_line.py gpurun_out/multirank.txt >/dev/null 2>&1
grep -o '"metric".\{0,160\}\|"parity": {[^}]*}\|"impl": "reference".\{0,80\}\|rror.\{0,200\}' gpurun_out/multirank.txt | head -20
