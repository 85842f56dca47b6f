"""PDL experiment: replay time per config with PDL off / on (early trigger)."""
import os, sys, pathlib, subprocess
ROOT = pathlib.Path(__file__).resolve().parent.parent
for early in (0, 1):
    for pdl in (0, 1):
        for cfg, b in ((3, 256), (3, 1), (1, 65536), (2, 1024), (0, 4096)):
            env = dict(os.environ, NNB_PDL=str(pdl))
            code = (f"import sys; sys.path.insert(0,'{ROOT}');"
                    f"from paper_1906_05737_b200 import kernels as K, EXACT, compile_model, zoo;"
                    f"o=K.Specializer.run\n"
                    f"def r(self):\n s=o(self); s.sources=['#define NNB_PDL_EARLY {early}\\n'+x for x in s.sources]; return s\n"
                    f"K.Specializer.run=r\n"
                    f"import torch; m,w=zoo.build({cfg}); net=compile_model(m,w,EXACT,batch={b},cache_dir='');"
                    f"net.apply(); torch.cuda.synchronize(); print(net.time_apply(iters=20))")
            out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
            print(f"early={early} pdl={pdl} cfg{cfg} b={b}: {out.stdout.strip()[:20]} ms {out.stderr[-200:] if out.returncode else ''}")
