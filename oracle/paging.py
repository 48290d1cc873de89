"""Deterministic slot + KV-page allocator restatement (TEST INFRASTRUCTURE ONLY).

Mirrors csrc/vox_api.cu (vox_admit / vox_release): lowest free slot; pages
popped from a LIFO free stack initialised so the first pops are 0,1,2,...;
ceil((prompt+target)/page_size) pages reserved at admission; release pushes a
request's pages back in reverse order (so a re-admission reuses them in the
same order).  The reference has no KV cache (profiles.py:318-331); the
contract is ours and the page tables are checked bit-exactly.
"""

from __future__ import annotations


class PageAllocator:
    def __init__(self, n_pages: int, page_size: int, max_slots: int):
        self.page_size = page_size
        self.free = list(range(n_pages - 1, -1, -1))
        self.used = [False] * max_slots
        self.pages: dict[int, list[int]] = {}

    def admit(self, prompt_len: int, target_len: int) -> int:
        slot = self.used.index(False)
        need = -(-(prompt_len + target_len) // self.page_size)
        if need > len(self.free):
            raise MemoryError("KV page pool exhausted")
        pages = [self.free.pop() for _ in range(need)]
        self.used[slot] = True
        self.pages[slot] = pages
        return slot

    def release(self, slot: int) -> None:
        for p in reversed(self.pages.pop(slot)):
            self.free.append(p)
        self.used[slot] = False

    def locate(self, slot: int, pos: int) -> tuple[int, int]:
        """(page, offset) of a token position: page_table[slot][pos // P], pos % P."""
        return self.pages[slot][pos // self.page_size], pos % self.page_size
