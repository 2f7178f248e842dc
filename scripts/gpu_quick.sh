#!/bin/bash
# quick GPU iteration: parity tests + C3 f32/u8 bench lines
mkdir -p gpurun_out
TAG=${TAG:-q}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; tail -5 gpurun_out/${TAG}_pytest.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/${TAG}_c3f32.json 2>gpurun_out/${TAG}_c3f32.err; cat gpurun_out/${TAG}_c3f32.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3f32', d['value'], d['ms_decode'], d['roofline']['frac'])"
timeout 300 python bench.py --no-cpu-baseline --out u8 > gpurun_out/${TAG}_c3u8.json 2>gpurun_out/${TAG}_c3u8.err; cat gpurun_out/${TAG}_c3u8.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3u8', d['value'], d['ms_decode'], d['roofline']['frac'])"
timeout 300 python bench.py --no-cpu-baseline --config c2_imagenet > gpurun_out/${TAG}_c2.json 2>gpurun_out/${TAG}_c2.err; cat gpurun_out/${TAG}_c2.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c2u8', d['value'], d['ms_decode'], d['roofline']['frac'])"
if [ -n "$NCU" ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:l3_decode_kernel -s 3 -c 1 -o gpurun_out/${TAG}_prof_c3f32 -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/${TAG}_ncu.log 2>&1
fi
