mkdir -p gpurun_out
for cfg in "1638 40 5120" "1638 2 256" "300 2 256"; do set -- $cfg
S=$1 H=$2 D=$3 python tools/debug_bins2.py /tmp/v2.npz; S=$1 H=$2 D=$3 KEEP_ATTN_V1=1 python tools/debug_bins2.py /tmp/v1.npz
python -c "
import numpy as np
a=np.load('/tmp/v1.npz'); b=np.load('/tmp/v2.npz')
S=a['s'].shape[0]
print('cfg $cfg: qts rel', np.abs(a['q']-b['q']).max()/np.abs(a['q']).max(), 'sts rel', np.abs(a['s']-b['s']).max()/np.abs(a['s']).max())
lt=np.tril_indices(S,-1)
print(' zeros v1', (a['s'][lt]==0).sum(), 'v2', (b['s'][lt]==0).sum(), 'sum', a['s'].sum(), b['s'].sum())
bad=np.argwhere(np.abs(a['s']-b['s'])>0.05*np.abs(a['s']).max()); print(' bad', len(bad), bad[:8].tolist())
"
done
