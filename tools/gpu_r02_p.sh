#!/bin/bash
# round 2, part P: ncu --set full of the bench kernel leg at every shape a bench line uses
# (roofline.traffic: DRAM bytes per launch), collected into profiles/ncu_kernel_traffic_r02.json
cd "$(dirname "$0")/.."
O=gpurun_out/p; mkdir -p $O
N="ncu --set full --clock-control none -k regex:(gemm_task|sgemm_tc2c) -s 1 -c 1"
timeout 600 $N -o $O/k_f64_2048 python tools/prof_kernel_leg.py 2048 2048 2048 f64 2 > $O/l1.log 2>&1
timeout 900 $N -o $O/k_f64_16384 python tools/prof_kernel_leg.py 16384 16384 16384 f64 2 > $O/l2.log 2>&1
timeout 900 $N -o $O/k_f64_16384_8192 python tools/prof_kernel_leg.py 16384 16384 8192 f64 2 > $O/l3.log 2>&1
timeout 1500 $N -o $O/k_f64_32768 python tools/prof_kernel_leg.py 32768 32768 32768 f64 2 > $O/l4.log 2>&1
timeout 900 $N -o $O/k_f32_32768 python tools/prof_kernel_leg.py 32768 32768 32768 f32 2 > $O/l5.log 2>&1
python tools/kernel_traffic.py $O/ncu_kernel_traffic_r02.json $O/k_f64_2048.ncu-rep:f64:2048x2048x2048 \
  $O/k_f64_16384.ncu-rep:f64:16384x16384x16384 $O/k_f64_16384_8192.ncu-rep:f64:16384x16384x8192 \
  $O/k_f64_32768.ncu-rep:f64:32768x32768x32768 $O/k_f32_32768.ncu-rep:f32:32768x32768x32768 > $O/collect.log 2>&1

for f in $O/k_*.ncu-rep; do python tools/ncu_summary.py $f > ${f%.ncu-rep}.txt 2>&1; done
rm -f $O/k_f64_2048.ncu-rep $O/k_f64_16384_8192.ncu-rep $O/k_f64_32768.ncu-rep $O/k_f32_32768.ncu-rep $O/k_f64_16384.ncu-rep
echo done > $O/status.txt
