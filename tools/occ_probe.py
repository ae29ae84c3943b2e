import sys, ctypes as C
sys.path.insert(0,'/root/repo')
import torch
from paper_2604_15272_b200 import population as P, plan as PL, _abi
torch.cuda.set_device(0); _abi.bind_device(0)
pop=P.load_population('G'); u=[x for x in P.units(pop) if x.cand.params=={'x':32,'i':1}][0]
for hints in [{}, {"max_cluster":4}]:
    p=PL.Plan(u.cand, 2, hints, 0); print(p.info['summary'][:160], p.info['smem_bytes'], p.info['threads'])
cuda=C.CDLL('libcuda.so.1')
# raw occupancy test of a trivial kernel with big dynamic smem via torch? use cudaOccupancy on a cupy-free path: skip
props=torch.cuda.get_device_properties(0)
print(props)
print('smem per SM', getattr(props,'shared_memory_per_multiprocessor',None), 'per block optin', getattr(props,'shared_memory_per_block_optin',None))
