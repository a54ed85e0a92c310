"""Input pipeline on the device: CIFAR-10 binary records, standardization and
flip / crop augmentation (drop-in for /root/reference/pkg/src/qtape/data.py).

The record files are read on the host (file I/O); everything after that runs
in the C-ABI kernels of csrc/data.cu on the GPU:

  * ``load_cifar10`` uploads the raw 3073-byte records once, decodes labels
    and fp32 pixels (u8 / 255) with qt_cifar_decode, takes the training
    split's per-channel mean / std with the float64 channel-moments kernel
    and standardizes in place with qt_standardize -- the dataset then stays
    resident in HBM (50 000 CIFAR images are 614 MB);
  * ``augment_batch`` / ``gather_batch`` draw the flips and crop offsets from
    the caller's numpy Generator with exactly the reference's calls
    (data.py:190-199), so a seeded run augments identically, and apply them
    with qt_gather_augment fused with the batch gather.

Bit-exactness: decode, standardize and augmentation are bit-identical to the
reference; the normalization constants are float64 moments in a fixed order
(numpy's pairwise order differs in the last bits; tests use a tolerance).
"""

from __future__ import annotations

import os
from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from . import _native as N
from .errors import DataError, FormatError

RECORD_BYTES = 3073                                   # data.py:20
TRAIN_FILES = [f"data_batch_{i}.bin" for i in range(1, 6)]
TEST_FILE = "test_batch.bin"
CROP_PAD = 4                                          # data.py:195


@dataclass
class Dataset:
    """images (N,C,H,W) float32 -- a CUDA tensor when loaded here, or a host
    array -- labels (N,) int64 on the host, as data.py:25-44."""

    images: object
    labels: np.ndarray
    num_classes: int
    norm_mean: Optional[np.ndarray] = None
    norm_std: Optional[np.ndarray] = None

    def __post_init__(self):
        self.labels = np.asarray(self.labels, dtype=np.int64)
        if len(self.images) != len(self.labels):
            raise DataError("images/labels length mismatch")
        if len(self.labels) and (self.labels.min() < 0 or self.labels.max() >= self.num_classes):
            raise DataError("label outside class range")

    def __len__(self) -> int:
        return len(self.labels)

    @property
    def on_device(self) -> bool:
        return isinstance(self.images, torch.Tensor) and self.images.is_cuda


def _read_records(path: str) -> np.ndarray:
    raw = np.fromfile(path, dtype=np.uint8)
    if raw.size == 0 or raw.size % RECORD_BYTES:
        raise FormatError(f"{path}: size {raw.size} is not a multiple of {RECORD_BYTES}")
    return raw.reshape(-1, RECORD_BYTES)


def load_cifar10(dir_path: str, split: str = "train", norm_stats: Optional[tuple] = None,
                 device=None) -> Dataset:
    """Load the CIFAR-10 binary batches under ``dir_path`` into HBM
    (data.py:60-87): partial training sets are accepted, the test split
    needs the training split's (mean, std)."""
    files = TRAIN_FILES if split == "train" else [TEST_FILE]
    paths = [os.path.join(dir_path, f) for f in files]
    present = [p for p in paths if os.path.exists(p)]
    if not present:
        raise FileNotFoundError(f"no {split} batch files under {dir_path}")
    if norm_stats is None and split != "train":
        raise DataError("test split needs norm_stats computed from the train split")
    rec = np.concatenate([_read_records(p) for p in present])
    n = rec.shape[0]
    dev = torch.device(device) if device is not None else \
        torch.device("cuda", torch.cuda.current_device())
    rec_d = torch.from_numpy(rec).to(dev)
    images = torch.empty((n, 3, 32, 32), dtype=torch.float32, device=dev)
    labels = torch.empty(n, dtype=torch.int64, device=dev)
    bad = torch.zeros(1, dtype=torch.int32, device=dev)
    N.call("qt_cifar_decode", N.ptr(rec_d), n, N.ptr(images), N.ptr(labels), N.ptr(bad))
    if int(bad.item()):
        raise DataError("CIFAR-10 label byte exceeds 9")
    del rec_d
    if norm_stats is None:
        from .ops import channel_moments
        m, v = channel_moments(images)
        mean = m.cpu().numpy()
        std = np.maximum(np.sqrt(v.cpu().numpy()), 1e-8)
    else:
        mean, std = (np.asarray(s, dtype=np.float64) for s in norm_stats)
    m32 = torch.from_numpy(mean.astype(np.float32)).to(dev)
    s32 = torch.from_numpy(std.astype(np.float32)).to(dev)
    N.call("qt_standardize", N.ptr(images), n, 3, 32 * 32, N.ptr(m32), N.ptr(s32))
    return Dataset(images=images, labels=labels.cpu().numpy(), num_classes=10,
                   norm_mean=np.asarray(mean), norm_std=np.asarray(std))


def write_cifar10_file(path: str, images_u8: np.ndarray, labels: np.ndarray) -> None:
    """(N,3,32,32) uint8 images + labels in the binary record layout (data.py:90-99)."""
    n = len(labels)
    if images_u8.shape != (n, 3, 32, 32) or images_u8.dtype != np.uint8:
        raise DataError("expected (N,3,32,32) uint8 images")
    out = np.empty((n, RECORD_BYTES), dtype=np.uint8)
    out[:, 0] = np.asarray(labels, dtype=np.uint8)
    out[:, 1:] = images_u8.reshape(n, -1)
    out.tofile(path)


def _class_grids(rng, classes: int, style: str) -> np.ndarray:
    """(K, 3, 8, 8) per-class level grids of the three corpus styles the
    reference's acceptance tests use (data.py:120-147): "smooth" uniform
    levels, "sparse" a dark field with five bright cells (heavy-tailed
    post-normalization activations), "natural" mid-range levels with four
    highlights (mild tails)."""
    if style == "smooth":
        return rng.uniform(40.0, 215.0, size=(classes, 3, 8, 8))
    if style not in ("sparse", "natural"):
        raise DataError(f"unknown style {style!r}")
    sparse = style == "sparse"
    grid = np.full((classes, 3, 8, 8), 25.0) if sparse else rng.uniform(40.0, 160.0, size=(classes, 3, 8, 8))
    for k in range(classes):
        for _ in range(5 if sparse else 4):
            ch, yy, xx = rng.integers(0, 3), rng.integers(0, 8), rng.integers(0, 8)
            if sparse:
                grid[k, ch, yy, xx] = 235.0
            else:
                grid[k, ch, yy, xx] += 140.0
    return grid


def synth_cifar_images(seed: int, n: int, classes: int = 10, noise: float = 32.0,
                       style: str = "bilinear"):
    """A learnable synthetic corpus in the CIFAR record format: every class
    is a random RGB pattern (an 8x8 grid of levels, upsampled to 32x32:
    bilinearly for the default "bilinear" style, as 4x4 blocks for the
    reference's "smooth" / "sparse" / "natural" styles), every sample that
    pattern cyclically shifted by up to 3 pixels plus Gaussian pixel noise,
    clipped to uint8.  The block styles draw the reference generator's
    random numbers in its order (data.py:114-165), so a seed gives the
    reference's corpus; "bilinear" is this package's own smooth variant."""
    rng = np.random.default_rng(seed)
    if style == "bilinear":
        grid = rng.uniform(40.0, 215.0, size=(classes, 3, 8, 8))
        t = (np.arange(32) + 0.5) / 4.0 - 0.5                # sample points on the 8x8 grid
        i0 = np.clip(np.floor(t).astype(int), 0, 7)
        i1 = np.clip(i0 + 1, 0, 7)
        f = np.clip(t - i0, 0.0, 1.0)
        rows = grid[:, :, i0, :] * (1 - f)[None, None, :, None] + grid[:, :, i1, :] * f[None, None, :, None]
        pat = rows[:, :, :, i0] * (1 - f) + rows[:, :, :, i1] * f          # (K,3,32,32)
    else:
        pat = _class_grids(rng, classes, style).repeat(4, axis=2).repeat(4, axis=3)
    labels = rng.permutation(np.arange(n) % classes).astype(np.int64)
    shift = rng.integers(-3, 4, size=(n, 2))             # (dy, dx) per sample
    imgs = np.stack([np.roll(pat[labels[i]], tuple(shift[i]), axis=(1, 2)) for i in range(n)])
    imgs = imgs + rng.standard_normal(imgs.shape) * noise
    return np.clip(imgs, 0, 255).astype(np.uint8), labels


def make_synthetic_cifar_dir(dir_path: str, seed: int = 0, train_n: int = 5000,
                             test_n: int = 1000, noise: float = 32.0,
                             style: str = "bilinear") -> str:
    """A synthetic corpus written in the CIFAR-10 binary layout, read back
    through the real parser (data.py:168-179)."""
    os.makedirs(dir_path, exist_ok=True)
    images, labels = synth_cifar_images(seed, train_n + test_n, noise=noise, style=style)
    write_cifar10_file(os.path.join(dir_path, TRAIN_FILES[0]), images[:train_n], labels[:train_n])
    write_cifar10_file(os.path.join(dir_path, TEST_FILE), images[train_n:], labels[train_n:])
    return dir_path


def augment_draws(n: int, rng: np.random.Generator, hflip: bool = True, translate: bool = True):
    """The reference's random draws for one batch, in its order
    (data.py:190-199): flips = rng.random(n) < 0.5, then the crop offsets
    rng.integers(0, 2 * 4 + 1, size=(n, 2))."""
    flips = rng.random(n) < 0.5 if hflip else None
    offs = rng.integers(0, 2 * CROP_PAD + 1, size=(n, 2)) if translate else None
    return flips, offs


def gather_batch(images: torch.Tensor, idx=None, rng: Optional[np.random.Generator] = None,
                 hflip: bool = True, translate: bool = True, out: Optional[torch.Tensor] = None,
                 n: Optional[int] = None) -> torch.Tensor:
    """out = augment(images[idx]) in one kernel (qt_gather_augment): the
    batch gather fused with the horizontal flip and the pad-4 random crop;
    without ``rng`` a plain gather."""
    if images.dim() != 4:
        raise DataError("augmentation expects a rank-4 batch")
    dev = images.device
    if idx is not None:
        idx_t = torch.as_tensor(np.asarray(idx, dtype=np.int64)).to(dev, non_blocking=True)
        n = len(idx)
    else:
        idx_t = None
        n = images.shape[0] if n is None else n
    c, h, w = images.shape[1:]
    flips = offs = None
    if rng is not None:
        f, o = augment_draws(n, rng, hflip, translate)
        if f is not None:
            flips = torch.from_numpy(f.astype(np.uint8)).to(dev, non_blocking=True)
        if o is not None:
            offs = torch.from_numpy(o.astype(np.int32)).to(dev, non_blocking=True)
    if out is None:
        out = torch.empty((n, c, h, w), dtype=torch.float32, device=dev)
    N.call("qt_gather_augment", N.ptr(images), N.ptr(idx_t), n, c, h, w, N.ptr(flips),
           N.ptr(offs), CROP_PAD, N.ptr(out))
    return out


def augment_batch(batch, rng: np.random.Generator, hflip: bool = True,
                  translate: bool = True):
    """Per-image horizontal flip (p = 0.5) and pad-4 random-crop translation
    (data.py:182-206) of a device batch; host arrays are uploaded first.
    Returns a new tensor; deterministic given the generator state."""
    if not isinstance(batch, torch.Tensor):
        arr = np.asarray(batch)
        if arr.ndim != 4:
            raise DataError("augmentation expects a rank-4 batch")
        batch = torch.from_numpy(np.ascontiguousarray(arr, dtype=np.float32)).cuda()
    N.require_cuda(batch, "batch")
    return gather_batch(batch.contiguous(), None, rng, hflip, translate)


def synth_blobs(seed: int, n: int, classes: int, shape, separation: float = 3.0,
                device=None) -> Dataset:
    """Gaussian clusters, balanced classes (data.py:100-116): class centres
    of norm ``separation`` in the flattened input space plus unit noise;
    the images are uploaded to the device."""
    if n < classes:
        raise DataError("need at least one sample per class")
    rng = np.random.default_rng(seed)
    shape = (shape,) if isinstance(shape, int) else tuple(shape)
    dim = int(np.prod(shape))
    centres = rng.standard_normal((classes, dim))
    centres *= separation / np.linalg.norm(centres, axis=1, keepdims=True)
    labels = np.arange(n) % classes
    rng.shuffle(labels)
    x = (centres[labels] + rng.standard_normal((n, dim))).reshape((n,) + shape).astype(np.float32)
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    return Dataset(images=torch.from_numpy(x).to(dev), labels=labels.astype(np.int64),
                   num_classes=classes)
