export CUDA_VISIBLE_DEVICES=0
timeout 900 python bench.py --seeds 5 --no-cpu-baseline > gpurun_out/seeds5.json 2>gpurun_out/seeds5.err; echo "rc=$?"; tail -3 gpurun_out/seeds5.err
python scripts/bsum.py gpurun_out/seeds5.json
python -c "
import json; d=json.loads([l for l in open('gpurun_out/seeds5.json').read().splitlines() if l.startswith('{')][-1]); print(d['seeds'], d['e2e']['value'], d['warmup'], d['steps'])"
