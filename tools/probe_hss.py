import sys; sys.path.insert(0, 'oracle/build'); sys.path.insert(0, 'tests')
import numpy as np
import _oracle as o
import paper_1611_01391_b200 as s
from hss_inputs import cauchy_kernel
M = cauchy_kernel(1024); B = M[512:640, 640:768]
I = [104, 10, 20, 124, 16, 23, 12, 11, 4, 30]
S = np.asfortranarray(B[I, :].T)
Q, _ = o.thin_qr(S)
print('oracle maxvol', o.maxvol_rows(Q, 1.1))
print('slra   maxvol', s.maxvol_rows(Q, 1.1))
print('oracle select', o.select_rows_spanning(S, 10, 1.1))
print('slra   select', s.select_rows_spanning(S, 10, 1.1))
Qs, _ = s.thin_qr(S)
print('Q diff', np.abs(np.abs(Qs) - np.abs(Q)).max())
