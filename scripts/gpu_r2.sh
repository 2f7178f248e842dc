#!/bin/bash
# round-2 GPU check: tests (all, or a -k subset via K=...), smoke, and the bench legs given in LEGS
mkdir -p gpurun_out
TAG=${TAG:-r2}
LEGS=${LEGS:-"c3f32 c1 compute ref"}
if [ -z "$NOTEST" ]; then
  timeout ${TEST_TIMEOUT:-1500} python -m pytest tests -m gpu -x -q ${K:+-k "$K"} > gpurun_out/${TAG}_pytest.log 2>&1; tail -5 gpurun_out/${TAG}_pytest.log
  timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; tail -1 gpurun_out/${TAG}_smoke.log
fi
summ() { python - "$1" <<'PY'
import json,sys
for ln in open(sys.argv[1]):
    if ln.startswith("{"):
        d=json.loads(ln); r=d.get("roofline") or {}
        print(sys.argv[1].split("/")[-1], d.get("value"), d.get("unit"), "ms_decode", d.get("ms_decode"), "frac", r.get("frac"), "e2e", (d.get("e2e") or {}).get("value"))
PY
}
for leg in $LEGS; do
  case $leg in
    c3f32) timeout 600 python bench.py $BENCH_ARGS > gpurun_out/${TAG}_c3f32.json 2> gpurun_out/${TAG}_c3f32.err ;;
    c3u8)  timeout 600 python bench.py --out u8 --no-cpu-baseline $BENCH_ARGS > gpurun_out/${TAG}_c3u8.json 2> gpurun_out/${TAG}_c3u8.err ;;
    c2)    timeout 600 python bench.py --config c2_imagenet --no-cpu-baseline $BENCH_ARGS > gpurun_out/${TAG}_c2.json 2> gpurun_out/${TAG}_c2.err ;;
    c4)    timeout 600 python bench.py --config c4_uhd --no-cpu-baseline $BENCH_ARGS > gpurun_out/${TAG}_c4.json 2> gpurun_out/${TAG}_c4.err ;;
    c1)    timeout 300 python bench.py --config c1_64x64 --steps 2000 --warmup 20 > gpurun_out/${TAG}_c1.json 2> gpurun_out/${TAG}_c1.err ;;
    compute) timeout 600 python bench.py --with-compute --steps 40 > gpurun_out/${TAG}_compute.json 2> gpurun_out/${TAG}_compute.err
             timeout 600 python bench.py --with-compute --steps 40 --max-ctas 296 > gpurun_out/${TAG}_compute_cap.json 2> gpurun_out/${TAG}_compute_cap.err ;;
    ref)   timeout 900 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/${TAG}_ref.json 2> gpurun_out/${TAG}_ref.err ;;
    two)   timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 20 --warmup 5 --share-device --dist-backend gloo --no-cpu-baseline > gpurun_out/${TAG}_two.json 2> gpurun_out/${TAG}_two.err ;;
  esac
  for f in gpurun_out/${TAG}_${leg}*.json; do summ $f; done
done
