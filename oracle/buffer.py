"""Token buffer O_i with KV-length and page accounting — the definition.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Follows Alg.1 ("Let O_i be token buffer for model i", P:97
"Rollback O_i to match O_j's last token", "Append matching tokens")
with the SPEC S:52-81 semantics and the stage-state notation of SURVEY.md §8:
tokens x[0..n-1] (prompt + committed), KV valid for positions 0..n-2, the
last token x[n-1] "pending" (its KV is computed by the next forward).

Paged KV accounting (§8(a) a12): a stage whose KV covers kv_len positions
holds ceil(kv_len / page_size) pages; a rollback frees the pages lying wholly
at or beyond the new kv_len.
"""
from __future__ import annotations


class ContractError(Exception):
    """keep > length etc. (SPEC S:77 — an engine bug, not a user error)."""


def pages_for(kv_len: int, page_size: int) -> int:
    return -(-kv_len // page_size)


class TokenBuffer:
    def __init__(self, tokens=()):
        self.tokens = list(map(int, tokens))
        self.kv_len = max(0, len(self.tokens) - 1)

    def __len__(self):
        return len(self.tokens)

    def append(self, toks) -> None:
        """Append tokens; the previous pending token and all but the last
        appended token get their KV written by the forward that produced them."""
        toks = list(map(int, toks))
        if not toks:
            return
        self.tokens.extend(toks)
        self.kv_len = len(self.tokens) - 1

    def rollback(self, keep: int) -> None:
        """O_i := O_i[0:keep]; kv_len := min(kv_len, keep-1); keep == len is a no-op."""
        if keep > len(self.tokens) or keep < 0:
            raise ContractError(f"rollback keep={keep} > length={len(self.tokens)}")
        self.tokens = self.tokens[:keep]
        self.kv_len = min(self.kv_len, max(keep - 1, 0))

    def resync(self, src) -> int:
        """Rollback to match src (reading R2): truncate to the first index
        where the tokens differ, then extend with src's suffix.  No-op when this
        buffer already extends src.  Returns the truncation point."""
        src = list(map(int, src))
        m = 0
        while m < min(len(src), len(self.tokens)) and src[m] == self.tokens[m]:
            m += 1
        if m == len(src):
            return len(self.tokens)          # already an extension of src
        self.rollback(m)
        self.tokens.extend(src[m:])
        # the resynced suffix has no KV yet: positions >= m-1 must be recomputed
        self.kv_len = min(self.kv_len, max(m - 1, 0))
        return m

    def pages(self, page_size: int) -> int:
        return pages_for(self.kv_len, page_size)
