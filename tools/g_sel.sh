timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
CMD="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-fft-comparator --streams 1"
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"mc_select|mc_scan|mc_rows|mc_units|iso_partial" -s 3 -c 6 --csv --log-file gpurun_out/gsel.csv $CMD > /dev/null 2>&1; echo ncu $?
