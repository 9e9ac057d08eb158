timeout 600 python tools/e2e_host_probe.py > gpurun_out/s36_e2e.txt 2>&1
CSVD_PROFILE_HOST=1 timeout 300 python -c "
import sys; sys.path.insert(0,'.')
import paper_2511_21702_b200 as P
from paper_2511_21702_b200 import workload as wl
T=wl.synth_vocab(128256,4096,64,0.3,1); ix=wl.fast_index(T,64,16)
q=wl.generate_queries(30,4096,'contextual',7,centroids=ix.centroids)
for h in q: P.decode_step(T,ix,h,P.DecodeConfig(k=10))
" 2> gpurun_out/s36_host_profile.txt > /dev/null
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k tie 2>&1 | tail -5 > gpurun_out/s36_pytest.txt
