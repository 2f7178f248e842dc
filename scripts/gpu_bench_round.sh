#!/bin/bash
# One gpurun session: bench lines for every config + ncu launch list + full ncu captures.
set -x
mkdir -p gpurun_out
TAG=${TAG:-r1}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${TAG}_smi.txt
timeout 600 python bench.py > gpurun_out/${TAG}_bench_c3_f32.json 2> gpurun_out/${TAG}_bench_c3_f32.err
timeout 600 python bench.py --out u8 --no-cpu-baseline > gpurun_out/${TAG}_bench_c3_u8.json 2> gpurun_out/${TAG}_bench_c3_u8.err
timeout 600 python bench.py --config c4_uhd --no-cpu-baseline > gpurun_out/${TAG}_bench_c4_u8.json 2> gpurun_out/${TAG}_bench_c4_u8.err
timeout 600 python bench.py --config c2_imagenet --no-cpu-baseline > gpurun_out/${TAG}_bench_c2_u8.json 2> gpurun_out/${TAG}_bench_c2_u8.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/${TAG}_bench_reference.json 2> gpurun_out/${TAG}_bench_reference.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_c3_f32.csv \
  python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/${TAG}_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:l3_decode_kernel -s 3 -c 1 \
  -o gpurun_out/${TAG}_prof_c3_f32 -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/${TAG}_ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:l3_decode_kernel -s 3 -c 1 \
  -o gpurun_out/${TAG}_prof_c3_u8 -f python bench.py --out u8 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/${TAG}_ncu_full_u8.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:l3_decode_kernel -s 3 -c 1 \
  -o gpurun_out/${TAG}_prof_c4_u8 -f python bench.py --config c4_uhd --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/${TAG}_ncu_full_c4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:l3_decode_kernel -s 3 -c 1 \
  -o gpurun_out/${TAG}_prof_c2_u8 -f python bench.py --config c2_imagenet --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/${TAG}_ncu_full_c2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:l3_decode_hwc_kernel -s 3 -c 1 \
  -o gpurun_out/${TAG}_prof_c3_f32_hwc -f python bench.py --crop 1024x2048 --layout hwc --out f32 --steps 3 --warmup 3 > gpurun_out/${TAG}_ncu_full_hwc.log 2>&1
timeout 600 python bench.py --ablation --config c3_cityscapes --steps 5 > gpurun_out/${TAG}_ablation_c3.json 2> gpurun_out/${TAG}_ablation_c3.err
for o in u8 f32; do for l in chw hwc; do
  timeout 300 python bench.py --crop 512x1024 --layout $l --out $o --steps 200 > gpurun_out/${TAG}_crop_c3_${o}_${l}.json 2> gpurun_out/${TAG}_crop_${o}_${l}.err
done; done
ls -la gpurun_out | grep ${TAG}
