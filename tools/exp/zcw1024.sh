# Z tile width at 1024 planes: 8 columns (1 CTA/SM) vs 4 columns (2 or 3 CTAs/SM), C5 single-GPU frame
for cw in 8 4; do
  VC_ZCW1024=$cw python bench.py --workload c5 --steps 20 --warmup 3 --no-cpu-baseline --no-fft-comparator > gpurun_out/zc_$cw.json 2> gpurun_out/zc_$cw.err; echo cw $cw $?
done
sed -i 's/^#define VC_Z1024_MINB 2/#define VC_Z1024_MINB 3/' paper_1712_03084_b200/csrc/k_fft.cu
(cd paper_1712_03084_b200/csrc && make -j32 > /dev/null 2>&1); echo build $?
VC_ZCW1024=4 python bench.py --workload c5 --steps 20 --warmup 3 --no-cpu-baseline --no-fft-comparator > gpurun_out/zc_4m3.json 2> gpurun_out/zc_4m3.err; echo cw4m3 $?
