"""The paper's three row-partition schemes, written out from §III (oracle side).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Plain Python, no shared
code with the product's ``mandel_plan_rows`` (C++), which the tests compare
against these functions.

Row indices are 0-based ("starting from the 0th index").
"""
from __future__ import annotations


def rows_per_task(height: int, n_tasks: int) -> int:
    """Eq. 16: rows per task = iYmax / number of tasks (floor)."""
    if n_tasks < 1:
        raise ValueError("n_tasks must be >= 1")
    return height // n_tasks


def naive_rows(height: int, n_tasks: int, rank: int) -> list[int]:
    """Naive row partition, Eq. 14, 15 and 17.

    S_r = (iYmax/N) * r                                   (Eq. 14)
    E_r = (iYmax/N) * (r + 1) - 1                          (Eq. 15; the printed
          "(r x 1)" is read as (r + 1), reading R12)
    E_r = E_r + (iYmax mod N) for the last rank r = N - 1  (Eq. 17)
    """
    if n_tasks < 1 or height < n_tasks or not 0 <= rank < n_tasks:
        raise ValueError("naive partition needs 1 <= N <= height and 0 <= rank < N")
    q = rows_per_task(height, n_tasks)
    s = q * rank
    e = q * (rank + 1) - 1
    if rank == n_tasks - 1:
        e = e + height % n_tasks
    return list(range(s, e + 1))


def alternating_rows(height: int, n_tasks: int, rank: int) -> list[int]:
    """Alternating row partition.

    "each node starts from their respective rank and increments with the number
    of tasks"; "In the case where the number of rows cannot be equally divided,
    the master node will then perform the remainder" -- the remainder rows are
    the ones past the last full round, [floor(H/N)*N, H), owned by rank 0.
    """
    if n_tasks < 1 or height < n_tasks or not 0 <= rank < n_tasks:
        raise ValueError("alternating partition needs 1 <= N <= height and 0 <= rank < N")
    full = rows_per_task(height, n_tasks) * n_tasks
    rows = list(range(rank, full, n_tasks))
    if rank == 0:
        rows += list(range(full, height))
    return rows


def fcfs_chunks(height: int, chunk_rows: int) -> list[list[int]]:
    """FCFS work units: the master hands out one row at a time
    "until the master node sends a row number larger than iYmax".  The GPU
    scheme hands out ``chunk_rows`` consecutive rows per claim (R13);
    chunk_rows = 1 is the paper's unit.  Returns the chunks in dispatch order."""
    if chunk_rows < 1:
        raise ValueError("chunk_rows must be >= 1")
    return [list(range(s, min(s + chunk_rows, height))) for s in range(0, height, chunk_rows)]


def message_count(scheme: str, height: int, n_tasks: int) -> int:
    """Eq. 18 (Naive, T_m = N - 1), Eq. 19 (FCFS, T_m = 2 iYmax), Eq. 20
    (Alternating, T_m = N - 1)."""
    if scheme in ("naive", "block"):
        return n_tasks - 1
    if scheme in ("alternating", "cyclic"):
        return n_tasks - 1
    if scheme == "fcfs":
        return 2 * height
    raise ValueError(scheme)
