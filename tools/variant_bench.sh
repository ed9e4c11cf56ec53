#!/bin/bash
# Build libholo_cuda with extra -D flags in a scratch copy and print the bench stage times.
# usage: tools/variant_bench.sh "<EXTRA_NVFLAGS>" <label>
set -e
src=$(pwd)
dst=/tmp/variant_$2
rm -rf $dst && cp -a $src $dst && cd $dst
touch paper_2506_08350_b200/csrc/${3:-composite}.cu
make -C paper_2506_08350_b200/csrc -j16 EXTRA_NVFLAGS="$1" > /dev/null
python bench.py --config ${CONFIG:-C3} --steps ${STEPS:-30} --warmup 5 --no-cpu-baseline --no-dropin --inflight ${INFLIGHT:-1} 2>/dev/null | python -c "
import json,sys; d=json.loads([l for l in sys.stdin.read().splitlines() if l.startswith('{')][-1]); print('$2', round(d['ms_per_step'],4), round(d['value'],1), {k: round(v['ms'],4) for k,v in d['stages'].items()})"
