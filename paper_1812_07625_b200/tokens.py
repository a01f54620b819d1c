"""Token table: the host-side id <-> symbol map the criterion adapters need.

Mirrors the reference's ``TokenTable`` (pkg/src/asrkit/lexicon.py:20-59):
the 0-based line number of a token file is the token id, ``<2>`` is the
ASG repetition token and ``|`` the word separator.
"""

from __future__ import annotations

from .errors import TokenError

REPETITION_SYMBOL = "<2>"


class TokenTable:
    def __init__(self, symbols):
        self.symbols = list(symbols)
        if not self.symbols:
            raise TokenError("token table is empty")
        self.ids = {}
        for i, sym in enumerate(self.symbols):
            if not sym:
                raise TokenError(f"empty token symbol at id {i}")
            if sym in self.ids:
                raise TokenError(f"duplicate token symbol {sym!r}")
            self.ids[sym] = i

    def __len__(self):
        return len(self.symbols)

    def __contains__(self, symbol):
        return symbol in self.ids

    def id(self, symbol: str) -> int:
        try:
            return self.ids[symbol]
        except KeyError:
            raise TokenError(f"unknown token symbol {symbol!r}") from None

    def symbol(self, token_id: int) -> str:
        if not 0 <= token_id < len(self.symbols):
            raise TokenError(f"token id {token_id} out of range 0..{len(self.symbols) - 1}")
        return self.symbols[token_id]

    @property
    def rep_id(self):
        """Id of the repetition token ``<2>``, or None (lexicon.py:50-54)."""
        return self.ids.get(REPETITION_SYMBOL)

    @property
    def silence_id(self):
        """Id of the word separator ``|``, or None (lexicon.py:56-59)."""
        return self.ids.get("|")


def load_tokens(path) -> TokenTable:
    """One symbol per line; trailing blank lines ignored (lexicon.py:62-67)."""
    with open(path, "r", encoding="utf-8") as f:
        symbols = [line.rstrip("\n") for line in f]
    while symbols and symbols[-1] == "":
        symbols.pop()
    return TokenTable(symbols)
