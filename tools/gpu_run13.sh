cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
python -c "
import torch; p=torch.cuda.get_device_properties(0); print('L2', p.L2_cache_size)
import ctypes; c=ctypes.CDLL('libcudart.so.12') if False else None
" 2>&1 | tail -1
for cfg in c4 c5; do
for v in "TPA_RELABEL=0" "TPA_RELABEL=1" "TPA_RELABEL=1 TPA_L2_PERSIST_MB=32" "TPA_RELABEL=1 TPA_L2_PERSIST_MB=64" "TPA_RELABEL=1 TPA_L2_PERSIST_MB=100"; do
  echo "== $cfg $v"; env $v python tools/ab_pre.py $cfg 2>&1 | tail -1 | grep -o "spmv.*ms [0-9.]*\|Error.*"
done
done
