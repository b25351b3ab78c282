cd /root/repo
bash tools/abv.sh ab30 "pre kc" "--config laplacian;--config laplacian --scale 0.3536;--config laplacian --scale 0.5;--config laplacian --scale 0.7071;--config banded27 --scale 0.3536" 2
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "parity or multichunk or kchunk" 2>&1 | tail -2
