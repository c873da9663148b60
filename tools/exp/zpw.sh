# windowed forward z-transforms at 256 planes: default vs VC_ZPW=0, alternating
python -m pytest tests -m gpu -x -q > gpurun_out/zpw_pytest.log 2>&1; echo pytest $?
for r in 1 2; do for v in 1 0; do
  VC_ZPW=$v python bench.py --steps 1000 --warmup 5 --no-cpu-baseline --no-fft-comparator > gpurun_out/zpw4_${v}_$r.json 2>&1; echo s4 $v $r $?
  VC_ZPW=$v python bench.py --steps 500 --warmup 5 --no-cpu-baseline --no-fft-comparator --streams 1 > gpurun_out/zpw1_${v}_$r.json 2>&1; echo s1 $v $r $?
done; done
