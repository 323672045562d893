"""The paper's worked example as ids (configs[0] of BASELINE.json).

Figure 1a triples: PAPER.md P:L29-L32.  Figure 2a query: P:L40-L45.

Entity / predicate id map.  The paper encodes "following the common practice"
(§6.2.1 step 2) without printing the map; the map below is the one
forced by Example 6.3's Mr array and first rows together with
Example 6.5's eliminated row 2 / column 3 and next-stage row sets
(P:L492-L502), unique up to a Product1<->Product2 swap (
DESIGN.md "Readings" R21).
"""
from .query import Query

ENTITY_IDS = {
    "User0": 0, "User1": 1, "Product0": 2, "User2": 3,
    "User3": 4, "User4": 5, "Product1": 6, "Product2": 7,
}
PREDICATE_IDS = {"follows": 1, "actor": 2, "director": 3, "FriendOf": 4}

# P:L29-L32, in the paper's order.
FIG1_TRIPLES_NAMED = [
    ("User0", "follows", "User1"), ("Product0", "actor", "User0"),
    ("Product0", "director", "User1"), ("Product0", "director", "User3"),
    ("Product0", "actor", "User4"), ("User3", "FriendOf", "User0"),
    ("User1", "follows", "User0"), ("Product1", "director", "User2"),
    ("Product1", "director", "User4"), ("User3", "follows", "User4"),
    ("User4", "follows", "User1"), ("Product2", "director", "User4"),
]

FIG1_N_ENTITIES = 8
FIG1_N_PREDICATES = 4


def fig1_triples():
    """(s, p, o) int lists of the 12 Fig. 1a triples under the id map above."""
    s = [ENTITY_IDS[a] for a, _, _ in FIG1_TRIPLES_NAMED]
    p = [PREDICATE_IDS[b] for _, b, _ in FIG1_TRIPLES_NAMED]
    o = [ENTITY_IDS[c] for _, _, c in FIG1_TRIPLES_NAMED]
    return s, p, o


def fig2_query() -> Query:
    """Fig. 2a: ?v0 actor ?v1 . ?v0 director ?v2 .
    ?v2 follows ?v1 . ?v3 follows ?v2 ."""
    a, d, f = PREDICATE_IDS["actor"], PREDICATE_IDS["director"], PREDICATE_IDS["follows"]
    return Query(vertices=(None, None, None, None),
                 edges=((0, a, 1), (0, d, 2), (2, f, 1), (3, f, 2)),
                 name="fig2")
