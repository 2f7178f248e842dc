bash scripts/micro/pipehalf.sh
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "predictor or config3 or c3 or fault" > gpurun_out/h2_pytest.log 2>&1; tail -3 gpurun_out/h2_pytest.log
for i in 1 2; do timeout 300 python bench.py --no-cpu-baseline --e2e-steps 2 > gpurun_out/h2_c3f32_$i.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/h2_c3f32_$i.json')); print('c3f32', d['value'], d['ms_decode'], d['roofline']['frac'])"; done
