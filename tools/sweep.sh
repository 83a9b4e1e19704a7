# usage: bash tools/sweep.sh "ENV=.. ENV2=.." ...   (one bench per setting, C2, 3 steps)
for s in "$@"; do
  env $s timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 1 > gpurun_out/sweep.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/sweep.json')); k=d['kernels_ms_per_step']
print('$s', round(d['ms_per_step'],2), {x: k.get(x) for x in ('build_search_kernel','beam_knn_kernel','build_prune_kernel','reverse_kernel')})"
done
