"""Oracle of Alg. 1, "Greedy Distribution Algorithm for ZeRO" (§2.3).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

    1: Sort T in descending order of their sizes -> T', C'
    2: Initialize memory usage u_j = 0 and partition p_j = {} for each GPU G_j
    3: for i = 1 to n:
    4:     j <- argmin_j u_j        (the GPU with the least memory usage)
    5:     p_j <- p_j U {(s'_i, t'_i)}
    6:     u_j <- u_j + c'_i
    8: return P = {p_1, ..., p_m}

Reading R21 (the algorithm leaves ties open): the sort is stable on the original
index (equal sizes keep ascending tensor index) and argmin takes the lowest device
index among equal loads.  Size c_i = number of elements (every
tensor of one state has the same element width, so bytes are proportional).
"""
from __future__ import annotations

from typing import List, Sequence, Tuple


def greedy_distribute(sizes: Sequence[int], m: int) -> Tuple[List[int], List[int], List[List[int]]]:
    """Returns (owner[t], load[j], partitions[j] as lists of original tensor indices)."""
    if m < 1:
        raise ValueError("m >= 1 required")
    order = sorted(range(len(sizes)), key=lambda i: (-sizes[i], i))        # line 1
    load = [0] * m                                                          # line 2
    parts: List[List[int]] = [[] for _ in range(m)]
    owner = [-1] * len(sizes)
    for i in order:                                                         # line 3
        j = min(range(m), key=lambda jj: (load[jj], jj))                    # line 4
        parts[j].append(i)                                                  # line 5
        owner[i] = j
        load[j] += sizes[i]                                                 # line 6
    return owner, load, parts
