#!/bin/bash
# k_gemm_tc: persistent grid sized to whole raster waves.  Tile t -> (j = t mod G, r = t div G) within a
# group and CTA c takes tiles c, c + grid, ...; with grid = 148 and G = 16 every wave (148 tiles =
# 9.25 r-tiles) splits one r-tile across two waves, so that X tile is fetched from DRAM twice (the
# CTAs sharing it are ~one tile apart); grid = 144 (G = 16) or 128 (G = 32 / 16) makes every wave
# whole r-tiles.  Under the 1000 W cap the 4 idle SMs may cost little.  Interleaved, c3 and c4.
O=gpurun_out/r02/wave; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for rep in 1 2 3; do
  for v in "16 0" "16 144" "32 128" "24 144" "16 128"; do
    set -- $v
    timeout 600 python bench.py --config c3 --raster-group $1 --max-ctas $2 --steps 20 --warmup 5 --e2e-steps 0 \
      --no-cpu-baseline > $O/c3_g$1_c$2_$rep.json 2>> $O/err.log
  done
done
for rep in 1 2; do
  for v in "16 0" "16 144" "32 128" "16 128"; do
    set -- $v
    timeout 600 python bench.py --config c4 --raster-group $1 --max-ctas $2 --steps 10 --warmup 3 --e2e-steps 0 \
      --no-cpu-baseline > $O/c4_g$1_c$2_$rep.json 2>> $O/err.log
  done
done
python - <<'PY'
import json, glob
for f in sorted(glob.glob('gpurun_out/r02/wave/*.json')):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, 'ERR', e); continue
    r = d['roofline']
    print(f.split('/')[-1], '%.4e' % d['value'], '%.3f ms' % r['avg_launch_ms'], d['clocks'].get('sm_mhz'), d['clocks'].get('power_w_max'))
PY
