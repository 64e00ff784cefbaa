import sys, numpy as np
sys.path.insert(0, ".")
import paper_1901_05128_b200 as fraq
from oracle.oracle import Oracle, ref_available
orc = Oracle("reference" if ref_available() else "port")
for g in (0.7, 0.3):
    w = np.array(fraq.sbd_weights(g, 1/65536, 65536).weights)
    ref = orc.sbd_weights(g, 1/65536, 65536)
    print(g, "sbd_weights n=65536 max rel", np.max(np.abs(w-ref)/np.maximum(np.abs(ref),1e-300)), "rel linf", np.max(np.abs(w-ref))/np.max(np.abs(ref)))
