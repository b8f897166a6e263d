# interleaved A/B of library builds on one config: bash scripts/r2_ab.sh CONFIG STEPS v2 v3 ...
c=$1; n=$2; shift 2
for rep in 1 2 3; do for v in "$@"; do
  TOPO_LIB_PATH=$PWD/paper_2005_05436_b200/_build/var/$v.so python bench.py --config $c --steps $n --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step'],4), {k:round(v,4) for k,v in d['stages_ms'].items()})"
done; done
