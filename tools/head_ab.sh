#!/bin/bash
# head split on/off at 1M documents of the config-3 and config-5 laws
OUT=gpurun_out/$1; mkdir -p $OUT
timeout 900 python -m pytest tests -x -q -m gpu -k "head or config_parity or stage1 or streaming" > $OUT/pytest.log 2>&1; echo "pytest $?" >> $OUT/status
for c in c3 c5; do for hd in 1 0; do
  SINN_HEAD=$hd SINN_DEBUG=$hd timeout 600 python bench.py --config $c --docs 1000000 --no-cpu-baseline --steps 5 --warmup 3 --e2e-steps 2 > $OUT/${c}_h$hd.json 2> $OUT/${c}_h$hd.err; echo "$c h$hd $?" >> $OUT/status
done; done
cat $OUT/status
