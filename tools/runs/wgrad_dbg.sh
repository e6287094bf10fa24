timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "wgrad_bias_building_block" 2>&1 | grep -E "assert|Error|error|rel_err" | head -20
python - <<'PY'
import numpy as np, torch, sys
sys.path.insert(0, '.')
import paper_2211_03578_b200 as tp
m = tp.TLP(tp.TLPConfig(precision="bf16"))
for (M,K,N) in [(32,32,32),(64,128,128),(2048,256,256)]:
    rng=np.random.default_rng(0)
    X=rng.normal(size=(M,K)).astype(np.float32); Y=rng.normal(size=(M,N)).astype(np.float32)
    out=torch.zeros(K*N+N,device='cuda')
    st=m.lib.tlp_debug_wgrad(m.h,M,K,N,torch.from_numpy(X).cuda().data_ptr(),K,torch.from_numpy(Y).cuda().data_ptr(),N,out.data_ptr(),torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    g=out.cpu().numpy(); W=g[:K*N].reshape(K,N); ref=X.T.astype(np.float64)@Y
    print(M,K,N,'st',st,'relW',np.abs(W-ref).max()/np.abs(ref).max(),'relb',np.abs(g[K*N:]-Y.sum(0)).max()/np.abs(Y.sum(0)).max())
    if M==32:
        np.set_printoptions(precision=2, linewidth=200)
        print(W[:4,:8]); print(ref[:4,:8])
        # try to identify permutation: correlate W rows/cols with ref
        R=ref
        for i in range(4):
            best=np.argmin([np.abs(W[i]-R[k]).max() for k in range(K)])
            print('row',i,'best ref row',best)
PY
