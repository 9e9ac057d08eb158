import sys, numpy as np
sys.path.insert(0, '.')
import paper_2511_21702_b200 as P
from paper_2511_21702_b200 import workload as wl, types as T
t = wl.synth_vocab(6, 5, 3, 0.4, 9, dtype="f64")
t = T.EmbeddingTable(weights=t.weights, bias=np.zeros(6))
r = P.dense_logits(t, np.ones(5)/np.sqrt(5))
print(r.logits)
