set -u
mkdir -p gpurun_out/r02
for mb in 128 256 512 1024; do echo "chunk_mb=$mb"; CGMIMO_CHUNK_MB=$mb python tools/quick_time.py cfg5 2>&1 | head -1; done
python -m pytest tests -m gpu -x -q --deselect tests/test_gpu_fullparity.py > gpurun_out/r02/gputest.log 2>&1; tail -3 gpurun_out/r02/gputest.log
python tests/parity_full.py --out gpurun_out/r02/parity.json > gpurun_out/r02/parity.log 2>&1; tail -3 gpurun_out/r02/parity.log
