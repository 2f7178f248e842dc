#!/bin/bash
# u8 narrow kernel on C3 (aligned, streamed) and C2 (mixed shapes, whole-staged)
python bench.py --crop 512x1024 --out u8 --steps 100 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C3 u8 narrow full', d['ms_full_decode'])"
python scripts/exp_c2_align.py
