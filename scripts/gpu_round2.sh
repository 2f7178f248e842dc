#!/bin/bash
# Round-2 measurement session (one gpurun call): bench lines for every config, the C1 latency line,
# the reference arm, the compute-concurrency legs, a 2-rank plumbing run, crop / HWC and ablation
# legs, the ncu launch list of a C3 step and ncu --set full captures of the decode kernels.
mkdir -p gpurun_out
TAG=${TAG:-r2}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${TAG}_smi.txt
run() { local name=$1; shift; timeout ${TO:-600} "$@" > gpurun_out/${TAG}_${name}.json 2> gpurun_out/${TAG}_${name}.err; tail -c 300 gpurun_out/${TAG}_${name}.json; echo; }
run bench_c3_f32 python bench.py
run bench_c3_u8 python bench.py --out u8 --no-cpu-baseline
run bench_c4_u8 python bench.py --config c4_uhd --no-cpu-baseline
run bench_c2_u8 python bench.py --config c2_imagenet --no-cpu-baseline
run latency_c1 python bench.py --config c1_64x64 --steps 2000 --warmup 20
run reference python bench.py --impl reference --steps 5 --warmup 1
run compute python bench.py --with-compute --steps 40
run compute_cap python bench.py --with-compute --steps 40 --max-ctas 296
TO=900 run two_ranks python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 2 --steps 20 --warmup 5 --share-device --dist-backend gloo --no-cpu-baseline
for o in u8 f32; do for l in chw hwc; do run crop_c3_${o}_${l} python bench.py --crop 512x1024 --layout $l --out $o --steps 200; done; done
run ablation_c3 python bench.py --ablation --config c3_cityscapes --steps 5
python scripts/exp_encoder.py > gpurun_out/${TAG}_encoder.jsonl 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_c3_f32.csv \
  python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/${TAG}_ncu_launch.log 2>&1
prof() { local key=$1 kern=$2; shift 2; timeout 900 ncu --set full --clock-control none --import-source on -k regex:$kern -s 3 -c 1 \
  -o gpurun_out/${TAG}_prof_${key} -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 "$@" > gpurun_out/${TAG}_ncu_${key}.log 2>&1; }
prof c3_f32 l3_decode_kernel
prof c3_u8 l3_decode_kernel --out u8
prof c4_u8 l3_decode_kernel --config c4_uhd
prof c2_u8 l3_decode_kernel --config c2_imagenet
ls -la gpurun_out | grep ${TAG}_ | wc -l
