"""Print the format of torch's CUDA IPC storage handle (dev probe for dist.peer_buffer)."""
import torch
from torch.multiprocessing.reductions import reduce_tensor
t = torch.empty((4, 64, 256, 4), device="cuda")
_, args = reduce_tensor(t)
h = args[7]
print("handle type", type(h), "len", len(h), "head", h[:12], "soff", args[9], "toff", args[3], "ssize", args[8])
print("expandable", torch.cuda.memory._get_current_allocator() if hasattr(torch.cuda.memory, "_get_current_allocator") else None)
