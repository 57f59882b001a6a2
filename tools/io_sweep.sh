# host staging sweep for the e2e path (diagnostic): threads x chunk x NT stores
for nt in 0 1; do for t in 4 8; do for ch in 1048576 4194304; do
echo "nt=$nt threads=$t chunk=$ch"; IMB_IO_NT=$nt IMB_IO_THREADS=$t IMB_IO_CHUNK=$ch IMB_TRACE=1 python tools/e2e_probe.py 2>&1 | grep -E "staged_h2d|step 2" | tail -2
done; done; done
