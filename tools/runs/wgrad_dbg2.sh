for d in 0 1 2; do
TLP_TMA_WGRAD_DEBUG=$d python - <<'PY'
import numpy as np, torch, sys, os
sys.path.insert(0, '.')
import paper_2211_03578_b200 as tp
m = tp.TLP(tp.TLPConfig(precision="bf16"))
M,K,N=32,32,32
rng=np.random.default_rng(0)
X=rng.normal(size=(M,K)).astype(np.float32); Y=rng.normal(size=(M,N)).astype(np.float32)
out=torch.zeros(K*N+N,device='cuda')
st=m.lib.tlp_debug_wgrad(m.h,M,K,N,torch.from_numpy(X).cuda().data_ptr(),K,torch.from_numpy(Y).cuda().data_ptr(),N,out.data_ptr(),torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
g=out.cpu().numpy(); W=g[:K*N].reshape(K,N); ref=X.T.astype(np.float64)@Y
np.set_printoptions(precision=2, linewidth=200, suppress=True)
print('dbg', os.environ['TLP_TMA_WGRAD_DEBUG'], 'relW', np.abs(W-ref).max()/np.abs(ref).max())
print(W[:3,:6]); print(ref[:3,:6])
PY
done
