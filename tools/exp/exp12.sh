timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -k "ragged or staged" 2>&1 | tail -3
timeout 2700 bash tools/profile_round.sh c3 c4 2>&1 | tail -20
ls -la gpurun_out/prof gpurun_out/prof_txt | head -40
du -sh gpurun_out
