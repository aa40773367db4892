import sys, ctypes, numpy as np
sys.path.insert(0,'.')
exec(open('tools/profile_cfg4.py').read())
lib=ctypes.CDLL('paper_2411_00546_b200/libocpgpu.so')
buf=(ctypes.c_ulonglong*8)()
lib.ocp_debug_phase(buf)
v=np.array(list(buf),dtype=float)
names=['','load','lu_aa','2b','2c','2d','update+writeout']
tot=v[1:7].sum()
for k in range(1,7): print(f"{names[k]:16s} {v[k]/tot*100:5.1f}%  {v[k]/ (256*391*8):9.0f} cyc/step")
print('warp_lu16 only', v[7]/(256*391*8))
