/*
 * ORACLE / TEST INFRASTRUCTURE ONLY — never linked into the product path.
 *
 * C restatement of the reference's sequential union-find kernel
 * `_uf_roots_py` (/root/reference/pkg/src/dendromst/contraction.py:53-73),
 * which the reference JIT-compiles with numba (:76-79).  Same algorithm,
 * same visiting order, same tie rule (the smaller root wins, :64-67), same
 * final flatten (:68-72), so the returned root array is identical.
 *
 * Built by oracle/Makefile into oracle/_build/liboracle.so and loaded by
 * oracle/dendro_oracle.py through ctypes.
 */
#include <stdint.h>

void oracle_uf_roots(int64_t num_vertices, int64_t num_edges,
                     const int64_t *cu, const int64_t *cv, int64_t *parent)
{
    for (int64_t x = 0; x < num_vertices; ++x) parent[x] = x;
    for (int64_t i = 0; i < num_edges; ++i) {
        int64_t a = cu[i];
        while (parent[a] != a) {          /* path halving, contraction.py:57-59 */
            parent[a] = parent[parent[a]];
            a = parent[a];
        }
        int64_t b = cv[i];
        while (parent[b] != b) {          /* contraction.py:61-63 */
            parent[b] = parent[parent[b]];
            b = parent[b];
        }
        if (a < b)                        /* contraction.py:64-67 */
            parent[b] = a;
        else if (b < a)
            parent[a] = b;
    }
    for (int64_t x = 0; x < num_vertices; ++x) {   /* flatten, contraction.py:68-72 */
        int64_t r = x;
        while (parent[r] != r) r = parent[r];
        parent[x] = r;
    }
}
