"""Print the error figures smoke() asserts on (development tool)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle as O
import paper_2603_08734_b200 as P
from paper_2603_08734_b200 import synth
from oracle import corpus  # noqa: E402
from paper_2603_08734_b200.device import DeviceCsr, build_device, spmm_device

a = corpus.generate_power_law(2048, 1536, 30000, 1.5, seed=1)
t = build_device(DeviceCsr.from_host(a))
b = torch.from_numpy(np.random.default_rng(2).uniform(-1, 1, (a.n_cols, 128)).astype(np.float32)).cuda()
ref32, ref64 = O.spmm_f64(O.Csr.of(a), b.cpu().numpy())
port = O.port_hybrid_spmm(O.build_format(O.Csr.of(a)), b.cpu().numpy()) if hasattr(O, "port_hybrid_spmm") else None
for v in (0, 64):
    c = spmm_device(t, b, math="fp32", cc_variant=v).cpu().numpy()
    print("variant", v, "fp32 max_rel", O.max_relative_error(c, ref32), "relF", O.rel_frobenius(c, ref64),
          "bitwise==port" if port is not None and np.array_equal(c, port) else "")
c = spmm_device(t, b, math="tf32").cpu().numpy()
print("tf32 relF", O.rel_frobenius(c, ref64))
m = P.build_rstile(a, P.split_long_work(a, P.partition_rows(a)))
cc = P.hybrid_spmm(m, P.DenseMatrix.from_array(b.cpu().numpy())).data
print("host api max_rel", O.max_relative_error(cc, ref32))
if port is not None:
    print("port max_rel", O.max_relative_error(port, ref32))
