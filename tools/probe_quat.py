import sys; sys.path.insert(0,'.')
import torch, json
from paper_2603_18695_b200 import capi, dev
from paper_2603_18695_b200.forge import op_info
op=capi.QUAT_F32; n=1<<27
ws=dev.Workspace(); src=dev.empty(op,n); dev.fill_synthetic(op,src,n,3); dst=dev.empty(op,n,"S")
for _ in range(3): dev.scan(op,True,src,dst,n,ws)
torch.cuda.synchronize()
a,b=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(10): dev.scan(op,True,src,dst,n,ws)
b.record(); torch.cuda.synchronize()
print(json.dumps({"quat_gbs": round(n*32/(a.elapsed_time(b)/10)/1e6,1)}))
