set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/g1_pytest.log 2>&1; echo pytest $?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g1_smoke.log 2>&1; echo smoke $?
timeout 600 python bench.py > gpurun_out/g1_bench.json 2> gpurun_out/g1_bench.err; echo bench $?
timeout 300 python bench.py --workload c3 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/g1_c3.json 2> gpurun_out/g1_c3.err; echo c3 $?
timeout 300 python bench.py --workload c5 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/g1_c5.json 2> gpurun_out/g1_c5.err; echo c5 $?
