"""Config-4 query set: large joins whose counts have closed forms (tests/closed_forms.py).

No method arithmetic here: only the query shapes.  Labels are data-vertex labels
of the config-4 graph (16 uniform labels), edges are wildcards.
"""
from .queries import Query

ANY = -1


def out_star(k, leaf_label=ANY, centre_label=ANY):
    return Query(k + 1, [centre_label] + [leaf_label] * k, [ANY] * (k + 1), [(0, i, ANY) for i in range(1, k + 1)])


def in_star(k, leaf_label=ANY, centre_label=ANY):
    return Query(k + 1, [centre_label] + [leaf_label] * k, [ANY] * (k + 1), [(i, 0, ANY) for i in range(1, k + 1)])


def path2(la=ANY, lb=ANY, lc=ANY):
    return Query(3, [la, lb, lc], [ANY] * 3, [(0, 1, ANY), (1, 2, ANY)])


# (name, query, mode): mode "match" writes every embedding, "count" counts the last level only
CFG4 = [
    ("out_star2_leaf0", out_star(2, leaf_label=0), "match"),
    ("in_star2_c0_leaf0", in_star(2, leaf_label=0, centre_label=0), "match"),
    ("path2_mid3", path2(ANY, 3, ANY), "match"),
    ("out_star3_c0_leaf0", out_star(3, leaf_label=0, centre_label=0), "count"),
]
