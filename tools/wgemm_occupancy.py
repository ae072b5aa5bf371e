"""Print the stream-K worker count the tcgen05 weight-contraction kernel would use (resident
CTA pairs) -- diagnostic."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
print(torch.cuda.get_device_properties(0))
