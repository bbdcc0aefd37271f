import time; t=time.time()
import sys; sys.path.insert(0,'.')
import numpy as np
import paper_2510_03421_b200 as P
t1=time.time(); a=np.random.rand(20,20)
P.glynn(a); t2=time.time(); P.glynn(a); t3=time.time()
P.ryser(a); t4=time.time(); P.opt(np.array([[1,2,3],[4,5,6],[7,8,9]])); t5=time.time()
print(f"import {t1-t:.3f}s first glynn {t2-t1:.3f}s second {1e6*(t3-t2):.1f}us first ryser {t4-t3:.3f}s first int opt {t5-t4:.3f}s")
