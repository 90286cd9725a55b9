"""Print how many clusters of the GEMM kernels can be co-resident (profiling helper)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2110_10221_b200 as P
print("SMs", P._lib.lib().cora_device_sm_count())
