# tests + C2 (S=4, S=1) + C5 lines
python -m pytest tests -m gpu -x -q > gpurun_out/ab_pytest.log 2>&1; echo pytest $?
python bench.py --steps 300 --warmup 5 --no-cpu-baseline --no-fft-comparator > gpurun_out/ab_b4.json 2>&1; echo b4 $?
python bench.py --steps 300 --warmup 5 --no-cpu-baseline --no-fft-comparator --streams 1 > gpurun_out/ab_b1.json 2>&1; echo b1 $?
python bench.py --workload c5 --steps 20 --warmup 3 --no-cpu-baseline --no-fft-comparator > gpurun_out/ab_c5.json 2>&1; echo c5 $?
