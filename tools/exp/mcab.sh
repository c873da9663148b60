python -m pytest tests -m gpu -x -q > gpurun_out/mc_pytest.log 2>&1; echo pytest $?
python bench.py --steps 200 --warmup 5 --no-cpu-baseline --no-fft-comparator > gpurun_out/mc_b4.json 2>&1; echo b4 $?
python bench.py --steps 200 --warmup 5 --no-cpu-baseline --no-fft-comparator --streams 1 > gpurun_out/mc_b1.json 2>&1; echo b1 $?
CMD="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-fft-comparator --streams 1"
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"mc_|iso_|ix_kernel" -s 40 -c 40 --csv --log-file gpurun_out/mcl.csv $CMD > gpurun_out/mcl.log 2>&1; echo l $?
