"""Workloads of BASELINE.json's configs: the models whose K-FAC layers the step
preconditions, synthetic data, and the per-layer factor shapes (M rows, a, g).

configs[0]  ResNet-20-style CIFAR net, 32x32, single worker (CPU reference runs it)
configs[1]  torchvision ResNet-50 v1.5, bs32/GPU, 224x224          (the bench workload)
configs[2]  same at 2/4/8 GPUs (fused factor all-reduce + LBP inverses)
configs[3]  DenseNet-201 (torchvision), bs16
configs[4]  Inception-v4 (`inceptionv4`, bs16, 299x299: 150 layers, non-square 1x7 / 7x1 kernels) and
            BERT-base linears: `bert_base_linears`, the 72 encoder linears of BERT-base at their
            real shapes (bs32 x seq128 = 4096 rows each) in a synthetic attention-free stack
"""

from __future__ import annotations

import torch
import torch.nn as nn


class _Basic(nn.Module):
    def __init__(self, cin, cout, stride):
        super().__init__()
        self.conv1 = nn.Conv2d(cin, cout, 3, stride, 1, bias=False)
        self.bn1 = nn.BatchNorm2d(cout)
        self.conv2 = nn.Conv2d(cout, cout, 3, 1, 1, bias=False)
        self.bn2 = nn.BatchNorm2d(cout)
        self.pad = cout - cin
        self.stride = stride

    def forward(self, x):
        out = torch.relu(self.bn1(self.conv1(x)))
        out = self.bn2(self.conv2(out))
        sc = x
        if self.stride != 1 or self.pad:  # option-A shortcut: subsample + zero-pad channels
            sc = x[:, :, ::self.stride, ::self.stride]
            sc = nn.functional.pad(sc, (0, 0, 0, 0, self.pad // 2, self.pad - self.pad // 2))
        return torch.relu(out + sc)


class ResNet20(nn.Module):
    """CIFAR ResNet-20 (He et al. 2016, option-A shortcuts): conv1 (a=27, g=16),
    18 3x3 convs, fc (a=64, g=10) -- 20 preconditioned layers."""

    def __init__(self, num_classes=10):
        super().__init__()
        self.conv1 = nn.Conv2d(3, 16, 3, 1, 1, bias=False)
        self.bn1 = nn.BatchNorm2d(16)
        blocks, cin = [], 16
        for cout, stride in ((16, 1), (32, 2), (64, 2)):
            for i in range(3):
                blocks.append(_Basic(cin, cout, stride if i == 0 else 1))
                cin = cout
        self.layers = nn.Sequential(*blocks)
        self.fc = nn.Linear(64, num_classes, bias=False)

    def forward(self, x):
        x = torch.relu(self.bn1(self.conv1(x)))
        x = self.layers(x)
        return self.fc(x.mean(dim=(2, 3)))


class _LinearBlock(nn.Module):
    """One BERT-base encoder layer's six linears (q, k, v, o: 768x768; ffn1 768->3072, ffn2
    3072->768) with post-LayerNorm residuals.  Attention's softmax mixing across tokens has no
    weights and is not preconditioned, so it is replaced by a per-token gate: the K-FAC work
    (factor rows, factor and gradient shapes) is that of BERT-base."""

    def __init__(self, h=768, f=3072):
        super().__init__()
        self.q, self.k, self.v, self.o = (nn.Linear(h, h, bias=False) for _ in range(4))
        self.ffn1 = nn.Linear(h, f, bias=False)
        self.ffn2 = nn.Linear(f, h, bias=False)
        self.ln1, self.ln2 = nn.LayerNorm(h), nn.LayerNorm(h)

    def forward(self, x):
        u = self.o(self.q(x) * torch.sigmoid(self.k(x)) + self.v(x))
        x = self.ln1(x + u)
        return self.ln2(x + self.ffn2(nn.functional.gelu(self.ffn1(x))))


class BertBaseLinears(nn.Module):
    """12 x _LinearBlock on synthetic [batch, seq, 768] token embeddings, mean-pooled into a
    768 -> 1000 classifier (73 preconditioned linears)."""

    def __init__(self, layers=12, num_classes=1000):
        super().__init__()
        self.blocks = nn.Sequential(*(_LinearBlock() for _ in range(layers)))
        self.fc = nn.Linear(768, num_classes, bias=False)

    def forward(self, x):
        return self.fc(self.blocks(x).mean(dim=1))


BERT_SEQ = 128


class _CBR(nn.Sequential):
    """conv (no bias) + BatchNorm + ReLU, the Inception unit; kernel / padding may be non-square."""

    def __init__(self, cin, cout, k, stride=1, pad=0):
        kk = k if isinstance(k, tuple) else (k, k)
        pp = pad if isinstance(pad, tuple) else (pad, pad)
        super().__init__(nn.Conv2d(cin, cout, kk, stride, pp, bias=False), nn.BatchNorm2d(cout, eps=1e-3),
                         nn.ReLU(inplace=False))


class _Branches(nn.Module):
    def __init__(self, *branches):
        super().__init__()
        self.b = nn.ModuleList(branches)

    def forward(self, x):
        return torch.cat([b(x) for b in self.b], 1)


class _Split(nn.Module):  # x -> cat(a(x), b(x)): the 1x3 / 3x1 pairs of Inception-C
    def __init__(self, a, b):
        super().__init__()
        self.a, self.b = a, b

    def forward(self, x):
        return torch.cat([self.a(x), self.b(x)], 1)


class InceptionV4(nn.Module):
    """Inception-v4 (Szegedy et al. 2016) on 299x299 inputs: the 149 convolutions + fc whose K-FAC
    factor dims the reference enumerates (profiles.py:346-405: 300 tensors, d 27..3456), including the
    non-square 1x7 / 7x1 / 1x3 / 3x1 kernels.  BASELINE.json configs[4]."""

    def __init__(self, num_classes=1000):
        super().__init__()
        C = _CBR
        mx = lambda: nn.MaxPool2d(3, 2)  # noqa: E731
        av = lambda: nn.AvgPool2d(3, 1, 1, count_include_pad=False)  # noqa: E731
        self.stem = nn.Sequential(
            C(3, 32, 3, 2), C(32, 32, 3), C(32, 64, 3, 1, 1),
            _Branches(mx(), C(64, 96, 3, 2)),                                                   # mixed3a: 160
            _Branches(nn.Sequential(C(160, 64, 1), C(64, 96, 3)),                                # mixed4a: 192
                      nn.Sequential(C(160, 64, 1), C(64, 64, (1, 7), 1, (0, 3)), C(64, 64, (7, 1), 1, (3, 0)),
                                    C(64, 96, 3))),
            _Branches(C(192, 192, 3, 2), mx()))                                                 # mixed5a: 384
        a = [_Branches(C(384, 96, 1), nn.Sequential(C(384, 64, 1), C(64, 96, 3, 1, 1)),
                       nn.Sequential(C(384, 64, 1), C(64, 96, 3, 1, 1), C(96, 96, 3, 1, 1)),
                       nn.Sequential(av(), C(384, 96, 1))) for _ in range(4)]
        ra = _Branches(C(384, 384, 3, 2), nn.Sequential(C(384, 192, 1), C(192, 224, 3, 1, 1), C(224, 256, 3, 2)), mx())
        b = [_Branches(C(1024, 384, 1),
                       nn.Sequential(C(1024, 192, 1), C(192, 224, (1, 7), 1, (0, 3)), C(224, 256, (7, 1), 1, (3, 0))),
                       nn.Sequential(C(1024, 192, 1), C(192, 192, (7, 1), 1, (3, 0)), C(192, 224, (1, 7), 1, (0, 3)),
                                     C(224, 224, (7, 1), 1, (3, 0)), C(224, 256, (1, 7), 1, (0, 3))),
                       nn.Sequential(av(), C(1024, 128, 1))) for _ in range(7)]
        rb = _Branches(nn.Sequential(C(1024, 192, 1), C(192, 192, 3, 2)),
                       nn.Sequential(C(1024, 256, 1), C(256, 256, (1, 7), 1, (0, 3)), C(256, 320, (7, 1), 1, (3, 0)),
                                     C(320, 320, 3, 2)), mx())
        c = [_Branches(C(1536, 256, 1),
                       nn.Sequential(C(1536, 384, 1), _Split(C(384, 256, (1, 3), 1, (0, 1)), C(384, 256, (3, 1), 1, (1, 0)))),
                       nn.Sequential(C(1536, 384, 1), C(384, 448, (3, 1), 1, (1, 0)), C(448, 512, (1, 3), 1, (0, 1)),
                                     _Split(C(512, 256, (1, 3), 1, (0, 1)), C(512, 256, (3, 1), 1, (1, 0)))),
                       nn.Sequential(av(), C(1536, 256, 1))) for _ in range(3)]
        self.features = nn.Sequential(*a, ra, *b, rb, *c)
        self.fc = nn.Linear(1536, num_classes, bias=False)

    def forward(self, x):
        x = self.features(self.stem(x))
        return self.fc(x.mean(dim=(2, 3)))


def build_model(name: str) -> nn.Module:
    import torchvision
    if name == "resnet50":
        return torchvision.models.resnet50(weights=None)
    if name == "resnet152":
        return torchvision.models.resnet152(weights=None)
    if name == "densenet201":
        return torchvision.models.densenet201(weights=None)
    if name == "resnet20":
        return ResNet20()
    if name == "bert_base_linears":
        return BertBaseLinears()
    if name == "inceptionv4":
        return InceptionV4()
    raise ValueError(f"unknown model {name!r}")


def input_shape(name: str, batch: int):
    if name == "bert_base_linears":
        return (batch, BERT_SEQ, 768)
    if name == "inceptionv4":
        return (batch, 3, 299, 299)
    return (batch, 3, 32, 32) if name == "resnet20" else (batch, 3, 224, 224)


def num_classes(name: str) -> int:
    return 10 if name == "resnet20" else 1000


def layer_shapes(name: str, batch: int) -> list:
    """[(layer name, M rows, a_dim, g_dim)] for every Conv2d/Linear in
    forward-definition order, M = batch * Hout * Wout (conv) or batch (linear)."""
    model = build_model(name)
    shapes = []
    hooks = []
    for n, m in model.named_modules():
        if isinstance(m, (nn.Conv2d, nn.Linear)):
            def hook(mod, inp, out, n=n):
                if isinstance(mod, nn.Conv2d):
                    a = mod.in_channels * mod.kernel_size[0] * mod.kernel_size[1]
                    shapes.append((n, batch * out.shape[2] * out.shape[3], a, mod.out_channels))
                else:
                    rows = batch * (inp[0].numel() // inp[0].shape[-1])  # probe runs at batch 1
                    shapes.append((n, rows, mod.in_features, mod.out_features))
            hooks.append(m.register_forward_hook(hook))
    with torch.no_grad():
        model.eval()(torch.zeros(input_shape(name, 1)))
    for h in hooks:
        h.remove()
    order = {n: i for i, (n, m) in enumerate(model.named_modules())}
    return sorted(shapes, key=lambda s: order[s[0]])


def bert_base_linear_shapes(batch: int = 32, seq: int = 128) -> list:
    """BERT-base encoder linears (12 layers x {q,k,v,o: 768x768, ffn 768->3072, 3072->768}); FC semantics."""
    m = batch * seq
    out = []
    for l in range(12):
        for nm in ("q", "k", "v", "o"):
            out.append((f"layer{l}.{nm}", m, 768, 768))
        out.append((f"layer{l}.ffn1", m, 768, 3072))
        out.append((f"layer{l}.ffn2", m, 3072, 768))
    return out
