import torch
p = torch.cuda.get_device_properties(0)
print(p.name, "L2", p.L2_cache_size)
import ctypes
rt = ctypes.CDLL("libcudart.so") if False else None
