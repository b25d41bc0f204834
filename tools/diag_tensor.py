import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2301_01179_b200 as g
geo = [(10.5, 10.5, 2.0), (16.5, 13.5, 3.0), (1.3, 0.7, 0.9)]
r, r1, x = (np.array(v) for v in zip(*geo))
T = g.tensor_batch(r, r1, x, 17, 8).cpu().numpy()
os.makedirs("gpurun_out", exist_ok=True)
np.save("gpurun_out/tensor_gpu_p8_K17.npy", T)
