for s in 2 1 3; do
  timeout 600 python bench.py --workload c5 --steps 40 --warmup 3 --no-cpu-baseline --streams $s > gpurun_out/c5s_$s.json 2> gpurun_out/c5s_$s.err; echo c5 S=$s $?
done
nvidia-smi --query-gpu=memory.used,memory.total --format=csv
