import sys, time, torch
sys.path.insert(0,'/root/repo')
from paper_2109_04131_b200.driver import Detector
from usfft_inputs import config
cfg=config(2); det=Detector(cfg)
t0=time.perf_counter(); I,_=det.run(); torch.cuda.synchronize(); t1=time.perf_counter()
I2,_=det.run(); torch.cuda.synchronize(); t2=time.perf_counter()
print("detect first %.1f ms, second %.1f ms" % (1e3*(t1-t0), 1e3*(t2-t1)))
for k in range(3):
    t0=time.perf_counter(); cov,coef=det.step3(I); torch.cuda.synchronize(); t1=time.perf_counter()
    print("step3 run %d: %.1f ms (lattices %d, M %d)" % (k, 1e3*(t1-t0), cov.z.shape[0], cov.M))
