import timeit, torch, ctypes, sys
sys.path.insert(0, '.')
import paper_2407_09577_b200 as fn
a = torch.empty(16, 4096, dtype=torch.bfloat16, device='cuda')
W = torch.empty(6144, 4096, dtype=torch.bfloat16, device='cuda')
z = torch.empty(16, 6144, dtype=torch.bfloat16, device='cuda')
n = 20000
def t(stmt, g=globals()):
    print(f"{stmt:60s} {1e6*timeit.timeit(stmt, number=n, globals=g)/n:.3f} us")
t("a.is_cuda"); t("a.is_contiguous()"); t("a.dim()"); t("a.shape[1]"); t("a.dtype == W.dtype"); t("a.device")
t("a.device == W.device"); t("a.data_ptr()"); t("torch.cuda.current_stream(a.device).cuda_stream")
t("torch._C._cuda_getCurrentRawStream(a.device.index)"); t("torch._C._cuda_getCurrentRawStream(0)")
t("fn._operands(a, W, 'linear')"); t("fn._out(z, 'out', (16, 6144), a.dtype, a.device)")
L = fn.lib()
f = L.flashnorm_linear_workspace_bytes
t("f(16, 4096, 6144, 0, 0, 0)")
t("tuple(z.shape) != (16, 6144)")
