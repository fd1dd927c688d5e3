# split-path chunk budget sweep on the headline config (run under gpurun)
for mb in 40 80 160 320 640; do
  echo "chunk_mb=$mb"; CGMIMO_CHUNK_MB=$mb python tools/quick_time.py cfg5 2>&1 | tail -2
done
python tools/quick_time.py cfg1 cfg2 cfg3 cfg4a_K2 cfg4a_K8 cfg4b_K2 cfg4b_K8 2>&1
