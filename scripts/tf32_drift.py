"""TF32 drift study (reading R8): one client's local SGD in torch fp32 with
the conv2 GEMM operands rounded to TF32 (RZ / RNA) vs fp64.  CPU only; minutes."""
import numpy as np, torch, torch.nn.functional as F, sys
sys.path.insert(0,'.'); import synth
torch.set_num_threads(8)
def q_rz(t):  # truncate fp32 to tf32 (drop 13 mantissa bits)
    i = t.float().contiguous().view(torch.int32); return (i & ~0x1FFF).view(torch.float32).to(t.dtype)
def q_rna(t):
    i = t.float().contiguous().view(torch.int32); return ((i + 0x1000) & ~0x1FFF).view(torch.float32).to(t.dtype)
class QConv(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, w, b, qa, qw):
        ctx.save_for_backward(x, w); ctx.qa, ctx.qw = qa, qw
        return F.conv2d(qa(x), qw(w), b, padding=2)
    @staticmethod
    def backward(ctx, g):
        x, w = ctx.saved_tensors
        gx = F.conv_transpose2d(ctx.qa(g), ctx.qw(w), padding=2)
        gw = torch.nn.grad.conv2d_weight(x, w.shape, g, padding=2)  # dW stays fp32 (SIMT)
        return gx, gw, g.sum((0,2,3)), None, None
ident = lambda t: t
def train(theta, x, y, mode, dtype, lr=0.05, B=32, steps=None):
    p, o = {}, 0
    for n, s in synth.param_shapes("cnn"):
        k=int(np.prod(s)); p[n]=torch.tensor(theta[o:o+k].reshape(s), dtype=dtype, requires_grad=True); o+=k
    qa, qw = {"exact":(ident,ident),"rz":(q_rz,q_rz),"rna_act":(q_rna,ident),"rna":(q_rna,q_rna)}[mode]
    n=len(y); X=torch.tensor(x,dtype=dtype).reshape(-1,3,32,32); Y=torch.tensor(y).long()
    for j in range(-(-n//B)):
        xb, yb = X[j*B:(j+1)*B], Y[j*B:(j+1)*B]
        h = F.max_pool2d(F.relu(F.conv2d(xb, p["conv1.w"], p["conv1.b"], padding=2)),2)
        h = F.max_pool2d(F.relu(QConv.apply(h, p["conv2.w"], p["conv2.b"], qa, qw)),2)
        h = F.relu(F.linear(h.flatten(1), p["fc1.w"], p["fc1.b"]))
        loss = F.cross_entropy(F.linear(h, p["fc2.w"], p["fc2.b"]), yb)
        g = torch.autograd.grad(loss, list(p.values()))
        with torch.no_grad():
            for t, gg in zip(p.values(), g): t -= lr*gg
    return np.concatenate([t.detach().double().numpy().ravel() for t in p.values()])
wl = synth.preset("C2"); theta = synth.init_params("cnn")
for n in [200, 600]:
    x, y = synth.client_data(wl, 7, n)
    ref = train(theta, x, y, "exact", torch.float64)
    for mode in ["exact", "rz", "rna_act", "rna"]:
        t = train(theta, x, y, mode, torch.float32)
        print(n, mode, "max|d| = %.2e" % np.max(np.abs(t-ref)), flush=True)

def traj(theta, x, y, lr, dtype, B=32):
    p, o = {}, 0
    for n_, s in synth.param_shapes("cnn"):
        k=int(np.prod(s)); p[n_]=torch.tensor(theta[o:o+k].reshape(s), dtype=dtype, requires_grad=True); o+=k
    n=len(y); X=torch.tensor(x,dtype=dtype).reshape(-1,3,32,32); Y=torch.tensor(y).long(); losses=[]
    for j in range(-(-n//B)):
        xb, yb = X[j*B:(j+1)*B], Y[j*B:(j+1)*B]
        h = F.max_pool2d(F.relu(F.conv2d(xb, p["conv1.w"], p["conv1.b"], padding=2)),2)
        h = F.max_pool2d(F.relu(F.conv2d(h, p["conv2.w"], p["conv2.b"], padding=2)),2)
        h = F.relu(F.linear(h.flatten(1), p["fc1.w"], p["fc1.b"]))
        loss = F.cross_entropy(F.linear(h, p["fc2.w"], p["fc2.b"]), yb); losses.append(loss.item())
        g = torch.autograd.grad(loss, list(p.values()))
        with torch.no_grad():
            for t, gg in zip(p.values(), g): t -= lr*gg
    return np.concatenate([t.detach().double().numpy().ravel() for t in p.values()]), losses

if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "--lr-sweep":
    # DESIGN.md reading R8: fp32-vs-fp64 divergence of one client's local SGD vs lr
    x, y = synth.client_data(wl, 7, 800)
    for lr in [0.05, 0.02, 0.01, 0.005]:
        a, _ = traj(theta, x, y, lr, torch.float64)
        b, _ = traj(theta, x, y, lr, torch.float32)
        print(f"lr={lr}: fp32-vs-fp64 max|d| = {np.max(np.abs(a - b)):.2e}")
