#!/bin/bash
# insert-path check: streaming/insert parity tests, config 4, and the default bench line (insert numbers)
TAG=${1:-ins}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests -x -q -m "gpu and not slow" -k "stream or insert or delete or recycl or compaction or config_parity or append" > $OUT/tests.log 2>&1; echo "tests $?" >> $OUT/status
timeout 1200 python bench.py --config c4 > $OUT/c4.json 2> $OUT/c4.err; echo "c4 $?" >> $OUT/status
timeout 900 python bench.py --steps 5 --warmup 3 --also none --no-cpu-baseline > $OUT/c5.json 2> $OUT/c5.err; echo "c5 $?" >> $OUT/status
cat $OUT/status
