"""Query-graph value type (§2.2.1: "each vertex corresponds
to a subject, object or variable and each edge corresponds to a predicate").

A `Query` is plain data:
  vertices : tuple, one entry per query vertex; ``None`` = variable,
             an ``int`` = constant entity id.
  edges    : tuple of (src, pred, dst) with src/dst vertex indices and
             pred a 1-based predicate id (a triple pattern src --pred--> dst).

Output columns of a query are its variable vertices in ascending vertex
index ("variable-index order"); a solution row lists their bindings in that
order.  This is a representation convention, not part of the method.
"""
from dataclasses import dataclass
from typing import Optional, Tuple


def var():
    return None


def const(entity_id: int):
    return int(entity_id)


@dataclass(frozen=True)
class Query:
    vertices: Tuple[Optional[int], ...]
    edges: Tuple[Tuple[int, int, int], ...]
    name: str = ""

    def __post_init__(self):
        object.__setattr__(self, "vertices", tuple(self.vertices))
        object.__setattr__(self, "edges", tuple(tuple(int(x) for x in e) for e in self.edges))

    @property
    def n_vertices(self) -> int:
        return len(self.vertices)

    @property
    def variables(self):
        """Vertex indices of variables, ascending (= output column order)."""
        return [i for i, v in enumerate(self.vertices) if v is None]

    def is_const(self, i: int) -> bool:
        return self.vertices[i] is not None

    def to_text(self) -> str:
        def t(i):
            v = self.vertices[i]
            return f"?v{i}" if v is None else f"<{v}>"
        pats = " . ".join(f"{t(s)} <p{p}> {t(o)}" for s, p, o in self.edges)
        sel = " ".join(f"?v{i}" for i in self.variables)
        return f"SELECT {sel} WHERE {{ {pats} }}"
