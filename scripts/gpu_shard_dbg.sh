cd $GRAFT_REPO_ROOT
export PYTHONFAULTHANDLER=1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=1 --master-addr 127.0.0.1 --master-port 29611 bench.py --sharded --steps 2 --warmup 3 --no-oracle 2>&1 | tail -30
echo "---- loopback"
timeout 300 python -c "
import torch, synth, time
from paper_2402_15253_b200 import sharded
import paper_2402_15253_b200 as pico
rp, ci = synth.CONFIGS['C2'].build(device=torch.device('cuda:0'))
for P in (1,2,4,8):
    torch.cuda.synchronize(); t=time.time()
    core, r, s = sharded.coreness_loopback(rp, ci, P); torch.cuda.synchronize()
    print('loopback P', P, 'ms %.1f'%((time.time()-t)*1e3), 'rounds', r, torch.equal(core, pico.coreness(rp, ci)))
" 2>&1 | tail -8
