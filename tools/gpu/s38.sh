timeout 900 python -m pytest tests/test_gpu_cluster.py -q -x 2>&1 | tail -15 > gpurun_out/s38_pytest.txt
timeout 900 python -c "
import sys, time; sys.path.insert(0,'.')
import paper_2511_21702_b200 as P
from paper_2511_21702_b200 import workload as wl
T=wl.synth_vocab(128256,4096,64,0.3,1)
t=time.time(); ix=P.build_index_gpu(T,1024,iters=8); print('c2 build_index_gpu (C=1024, 8 iters):', round(time.time()-t,1),'s', ix.n_clusters)
q=wl.generate_queries(3,4096,'contextual',7,centroids=ix.centroids)
for h in q:
    o=P.decode_step(T,ix,h,P.DecodeConfig(k=10)); print(o.status.kind, o.fallback_used, o.stats.clusters_opened, o.stats.sub_size)
" > gpurun_out/s38_build.txt 2>&1
