import sys, torch
sys.path.insert(0, '.')
import __graft_entry__ as g
g.smoke()
import paper_2403_08245_b200 as sm
torch.manual_seed(0)
T, d, de, E, k = 512, 256, 512, 8, 2
x = (torch.rand(T, d, device='cuda')*2-1).bfloat16(); dy = (torch.rand(T, d, device='cuda')*2-1).bfloat16()
w1 = ((torch.rand(E, d, de, device='cuda')*2-1)/16).bfloat16(); w2 = ((torch.rand(E, de, d, device='cuda')*2-1)/23).bfloat16()
r = sm.topk_select(torch.softmax(torch.randn(T, E, device='cuda'), 1), k)
o = sm.compute_grouped_order(r)
y, ctx = sm.smoe_mlp_forward(x, w1, w2, r, o); gr = sm.smoe_mlp_backward(ctx, dy)
yi = sm.smoe_mlp_forward(x, w1, w2, r, o, training=False)
torch.cuda.synchronize(); print('ok')
