mkdir -p gpurun_out/r3u
FTAR_PDL_EARLY=2 timeout 900 python -m pytest tests/test_gpu_multiproc.py -q -x -k "queued_calls" > gpurun_out/r3u/t.log 2>&1
echo done
