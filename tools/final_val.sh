# Round-end validation on one B200: smoke, GPU suite, the default bench line,
# the reference arm, the data-parallel learner, one Catch acceptance seed.
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; tail -1 gpurun_out/bench_default.json | cut -c1-400
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; tail -1 gpurun_out/bench_ref.json | cut -c1-300
timeout 600 python bench.py --mode dp --steps 300 --warmup 5 --no-cpu > gpurun_out/bench_dp.json 2> gpurun_out/bench_dp.err; tail -1 gpurun_out/bench_dp.json | cut -c1-300
timeout 600 python tools/catch_acceptance.py gpurun_out/catch_final 1 > gpurun_out/catch.log 2>&1; tail -2 gpurun_out/catch.log
