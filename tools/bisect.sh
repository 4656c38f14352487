for k in 4 8 16 32; do
  echo "== dbg=$k"
  RPC_DEBUG_UPDATE=$k RPC_DEBUG_SYNC=1 timeout 120 python -c "
import sys; sys.path.insert(0,'.'); sys.path.insert(0,'oracle')
from paper_2410_03969_b200 import api, workloads as wl
x = wl.gen_c1(4000, 10, 0)
try:
    r = api.accelerated_rpcholesky(api.KernelOracle(x, api.KernelSpec('gaussian', 3.16)), api.RunConfig.until_rank(200, 40, 0))
    print('ok rank', r.rank)
except Exception as e: print('ERR', e)
" 2>&1 | tail -2
done
