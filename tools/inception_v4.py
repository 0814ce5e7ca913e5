"""Inception-v4 (Szegedy et al., AAAI 2017, "Inception-v4, Inception-ResNet
and the Impact of Residual Connections on Learning", Figures 3-9) for the
trace extraction and the real-training bench (tools only; torchvision has no
Inception-v4). The paper's Table 3 (reference PAPER.md:597-604) lists it with
449 tensors and ~42.6 M parameters: 149 convolutions, each conv (no bias) +
BatchNorm (gamma, beta) = 3 tensors, plus the classifier weight and bias.
"""
from __future__ import annotations

import torch
from torch import nn


class Conv(nn.Sequential):
    """conv (no bias) -> BN -> ReLU; 3 parameter tensors."""

    def __init__(self, cin, cout, k, s=1, p=0):
        super().__init__(nn.Conv2d(cin, cout, k, stride=s, padding=p, bias=False),
                         nn.BatchNorm2d(cout, eps=1e-3), nn.ReLU(inplace=True))


class Cat(nn.Module):
    """Run the branches on one input and concatenate along channels."""

    def __init__(self, *branches):
        super().__init__()
        self.branches = nn.ModuleList(branches)

    def forward(self, x):
        return torch.cat([b(x) for b in self.branches], 1)


def _pool_proj(cin, cout):
    return nn.Sequential(nn.AvgPool2d(3, 1, 1, count_include_pad=False), Conv(cin, cout, 1))


class Stem(nn.Sequential):
    """Figure 3: 3 -> 384 channels."""

    def __init__(self):
        super().__init__(
            Conv(3, 32, 3, 2), Conv(32, 32, 3), Conv(32, 64, 3, p=1),
            Cat(nn.MaxPool2d(3, 2), Conv(64, 96, 3, 2)),
            Cat(nn.Sequential(Conv(160, 64, 1), Conv(64, 96, 3)),
                nn.Sequential(Conv(160, 64, 1), Conv(64, 64, (1, 7), p=(0, 3)), Conv(64, 64, (7, 1), p=(3, 0)),
                              Conv(64, 96, 3))),
            Cat(Conv(192, 192, 3, 2), nn.MaxPool2d(3, 2)),
        )


def inception_a():  # Figure 4: 384 -> 384
    return Cat(Conv(384, 96, 1),
               nn.Sequential(Conv(384, 64, 1), Conv(64, 96, 3, p=1)),
               nn.Sequential(Conv(384, 64, 1), Conv(64, 96, 3, p=1), Conv(96, 96, 3, p=1)),
               _pool_proj(384, 96))


def reduction_a():  # Figure 7 (k, l, m, n = 192, 224, 256, 384): 384 -> 1024
    return Cat(Conv(384, 384, 3, 2),
               nn.Sequential(Conv(384, 192, 1), Conv(192, 224, 3, p=1), Conv(224, 256, 3, 2)),
               nn.MaxPool2d(3, 2))


def inception_b():  # Figure 5: 1024 -> 1024
    return Cat(Conv(1024, 384, 1),
               nn.Sequential(Conv(1024, 192, 1), Conv(192, 224, (1, 7), p=(0, 3)), Conv(224, 256, (7, 1), p=(3, 0))),
               nn.Sequential(Conv(1024, 192, 1), Conv(192, 192, (7, 1), p=(3, 0)), Conv(192, 224, (1, 7), p=(0, 3)),
                             Conv(224, 224, (7, 1), p=(3, 0)), Conv(224, 256, (1, 7), p=(0, 3))),
               _pool_proj(1024, 128))


def reduction_b():  # Figure 8: 1024 -> 1536
    return Cat(nn.Sequential(Conv(1024, 192, 1), Conv(192, 192, 3, 2)),
               nn.Sequential(Conv(1024, 256, 1), Conv(256, 256, (1, 7), p=(0, 3)), Conv(256, 320, (7, 1), p=(3, 0)),
                             Conv(320, 320, 3, 2)),
               nn.MaxPool2d(3, 2))


class InceptionC(nn.Module):  # Figure 6: 1536 -> 1536
    def __init__(self):
        super().__init__()
        self.b0 = Conv(1536, 256, 1)
        self.b1 = Conv(1536, 384, 1)
        self.b1a = Conv(384, 256, (1, 3), p=(0, 1))
        self.b1b = Conv(384, 256, (3, 1), p=(1, 0))
        self.b2 = nn.Sequential(Conv(1536, 384, 1), Conv(384, 448, (3, 1), p=(1, 0)), Conv(448, 512, (1, 3), p=(0, 1)))
        self.b2a = Conv(512, 256, (1, 3), p=(0, 1))
        self.b2b = Conv(512, 256, (3, 1), p=(1, 0))
        self.b3 = _pool_proj(1536, 256)

    def forward(self, x):
        y1, y2 = self.b1(x), self.b2(x)
        return torch.cat([self.b0(x), self.b1a(y1), self.b1b(y1), self.b2a(y2), self.b2b(y2), self.b3(x)], 1)


class InceptionV4(nn.Module):
    def __init__(self, num_classes: int = 1000):
        super().__init__()
        self.features = nn.Sequential(Stem(), *[inception_a() for _ in range(4)], reduction_a(),
                                      *[inception_b() for _ in range(7)], reduction_b(),
                                      *[InceptionC() for _ in range(3)])
        self.pool = nn.AdaptiveAvgPool2d(1)
        self.drop = nn.Dropout(0.2)
        self.fc = nn.Linear(1536, num_classes)

    def forward(self, x):
        return self.fc(self.drop(torch.flatten(self.pool(self.features(x)), 1)))


def inception_v4(num_classes: int = 1000) -> InceptionV4:
    return InceptionV4(num_classes)


if __name__ == "__main__":
    m = inception_v4()
    ps = [p for p in m.parameters() if p.requires_grad]
    print(len(ps), sum(p.numel() for p in ps))
    print(m(torch.randn(2, 3, 224, 224)).shape)
