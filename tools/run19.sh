cd /root/repo
for A in "--config rmat --reorder" "--config rmat"; do
for E in "DTANS_LONG_SEG=64" "DTANS_LONG_SEG=0" "DTANS_LONG_SEG=2" "DTANS_LONG_SEG=4" "DTANS_LONG_SEG=8" "DTANS_LONG_SEG=16" "DTANS_LONG_SEG=0 DTANS_CHUNK=32" "DTANS_LONG_SEG=4 DTANS_CHUNK=32"; do
    echo "$E $A $(env $E timeout 900 python tools/kbench.py $A --cache /tmp/kbc 2>&1 | tail -1 | cut -c90-400)"
done
done
