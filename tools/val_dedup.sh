mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_frame_ring.py -q 2>&1 | tail -1
timeout 300 python tools/dedup_learner_check.py 2>&1 | tail -2
timeout 600 python tools/kernel_bench.py gpurun_out/kernel_bench.json > gpurun_out/kb.log 2>&1; grep -E "ring_gather|frame_dedup" gpurun_out/kb.log | cut -c1-200
