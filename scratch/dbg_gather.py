import sys, ctypes as C, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from oracle import oracle as O
from paper_2305_03152_b200 import vipkit as vk
from conftest import csr_from
import numpy as np
g = dict(np.load('/root/repo/tests/golden/graphs.npz')); fx = dict(np.load('/root/repo/tests/golden/expand_grid.npz'))
port = O.port()
csr = csr_from(g, 'pa5000')
import test_gpu_plane as T
r = T._pipeline(vk, port, csr, fx['roles'], fx['labels'], 4, [15,10,5], 64, 0.2, 42, 64, 0, 1234, 3)
print(r['counts'])
s = r['sampler']; fs, ec, al = s.sizes(); print('all sizes', al)
