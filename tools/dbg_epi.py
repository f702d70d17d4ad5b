import sys, subprocess
sys.path.insert(0, '.')
CASES = {
 "mask_k1": "conv.conv_dgrad(dy, wd, (n,t,h,w,cin), mask=m)",
 "mask_k3": "conv.conv_dgrad(dy3, wd3, (n,t,h,w,cin), k=3, mask=m)",
 "res_k1": "conv.conv_dgrad(dy, wd, (n,t,h,w,cin), residual=m)",
 "shift32_nores": "conv.conv_dgrad(dy, wd, (n,t,h,w,cin), fold=(32,32))",
 "shift32_res": "conv.conv_dgrad(dy, wd, (n,t,h,w,cin), fold=(32,32), residual=m)",
}
if len(sys.argv) == 1:
    for k in CASES:
        r = subprocess.run([sys.executable, __file__, k], capture_output=True, text=True)
        print(k, "OK" if r.returncode == 0 else "FAIL: " + (r.stderr.strip().splitlines() or ["?"])[-1])
    sys.exit(0)
import torch
from paper_1910_00932_b200 import conv
n,t,h,w,cin,cout = 1,4,6,6,256,64
dy = torch.randn(n,t,h,w,cout,device='cuda').bfloat16()
dy3 = torch.randn(n,t,h,w,cout,device='cuda').bfloat16()
wd = torch.randn(cin,1,1,cout,device='cuda').bfloat16()
wd3 = torch.randn(cin,3,3,cout,device='cuda').bfloat16()
m = torch.randn(n,t,h,w,cin,device='cuda').bfloat16()
out = eval(CASES[sys.argv[1]])
torch.cuda.synchronize()
