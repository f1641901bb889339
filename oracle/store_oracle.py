"""TEST INFRASTRUCTURE — numpy restatement of streamcut/store.py (the checker
for the GPU partitioned-storage path, never the product).

  buckets(edges, labels)          store.py:55-104 (write_buckets): bucket id
                                  label[u] * p + label[v], p = 1 + max label
                                  >= 0; a stable sort by bucket id keeps the
                                  input order inside a bucket (store.py:92-94)
  bucket_file_bytes(...)          the store file + .idx sidecar bytes
  grouping(labels)                store.py:221-227 (reorder_features): stable
                                  argsort by label, its inverse, extents

Pinned against the real reference by tests/golden/golden_store.json
(tests/golden/make_golden_store.py runs streamcut itself).
"""
import struct

import numpy as np


def buckets(edges, labels):
    e = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
    lab = np.asarray(labels, dtype=np.int64)
    assigned = lab[lab >= 0]
    p = int(assigned.max()) + 1 if assigned.size else 1
    if e.shape[0]:
        lu, lv = lab[e[:, 0]], lab[e[:, 1]]
        if (lu < 0).any() or (lv < 0).any():
            raise ValueError("unlabeled endpoint encountered")
        key = lu * p + lv
    else:
        key = np.zeros(0, dtype=np.int64)
    order = np.argsort(key, kind="stable")
    counts = np.bincount(key, minlength=p * p) if key.size else np.zeros(p * p, dtype=np.int64)
    return p, e[order], counts.astype(np.int64)


def bucket_file_bytes(edges, labels, width=32):
    p, grouped, counts = buckets(edges, labels)
    pair = 2 * (width // 8)
    head = struct.pack("<4sIIIQ", b"GRPB", 1, p, 1 if width == 64 else 0, int(counts.sum()))
    body = grouped.astype("<u8" if width == 64 else "<u4").tobytes()
    starts = np.concatenate([[0], np.cumsum(counts)[:-1]]) if counts.size else np.zeros(0, np.int64)
    side = np.empty((p * p, 2), dtype="<u8")
    side[:, 0] = struct.calcsize("<4sIIIQ") + starts * pair
    side[:, 1] = counts
    return head + body, side.tobytes()


def grouping(labels):
    lab = np.asarray(labels, dtype=np.int64)
    n = lab.shape[0]
    order = np.argsort(lab, kind="stable")
    perm = np.empty(n, dtype=np.int64)
    perm[order] = np.arange(n)
    p = int(lab.max()) + 1 if n else 1
    counts = np.bincount(lab, minlength=p)
    starts = np.concatenate([[0], np.cumsum(counts)[:-1]])
    return order, perm, tuple((int(s), int(c)) for s, c in zip(starts, counts))
