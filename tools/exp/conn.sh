# root branch on/off x CUDA_DEVICE_MAX_CONNECTIONS default/32, S=4 and S=1
for rb in 1 0; do for conn in 8 32; do
  CUDA_DEVICE_MAX_CONNECTIONS=$conn VC_ROOT_BRANCH=$rb python bench.py --steps 1000 --warmup 5 --no-cpu-baseline --no-fft-comparator > gpurun_out/cn4_${rb}_$conn.json 2>&1; echo s4 rb=$rb conn=$conn $?
  CUDA_DEVICE_MAX_CONNECTIONS=$conn VC_ROOT_BRANCH=$rb python bench.py --steps 500 --warmup 5 --no-cpu-baseline --no-fft-comparator --streams 1 > gpurun_out/cn1_${rb}_$conn.json 2>&1; echo s1 rb=$rb conn=$conn $?
done; done
