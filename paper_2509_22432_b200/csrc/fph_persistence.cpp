// fph_persistence.cpp -- Z/2 boundary-matrix reduction with the twist
// (clearing) optimisation, host C++.
//
// Same contract as reference floodph/persistence.py:89 _run_reduction and
// :118 reduce_and_extract: columns in filtration order, each column the
// sorted ranks of its facets; dimensions processed top-down, a column whose
// index is already a pivot is cleared; a column is reduced by adding the
// column that owns its lowest row until the lowest row is unowned or the
// column is empty.  The persistence pairing does not depend on the order of
// column additions, so the pairs (and the diagram) equal the reference's.
// The north star keeps this stage on the host; this file only makes it fast.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <vector>

#include "../../include/floodph_b200.h"

namespace fph {
void set_error(const char* fmt, ...);
}

namespace {

// a ^= b for strictly increasing index lists, into out
void sym_diff(const std::vector<int32_t>& a, const std::vector<int32_t>& b,
              std::vector<int32_t>& out) {
    out.clear();
    size_t i = 0, j = 0;
    while (i < a.size() && j < b.size()) {
        if (a[i] == b[j]) {
            ++i;
            ++j;
        } else if (a[i] < b[j]) {
            out.push_back(a[i++]);
        } else {
            out.push_back(b[j++]);
        }
    }
    out.insert(out.end(), a.begin() + i, a.end());
    out.insert(out.end(), b.begin() + j, b.end());
}

}  // namespace

extern "C" int fph_persistence_pairs(int32_t max_dim, const int64_t* counts,
                                     const int32_t* const* facets, const int64_t* order,
                                     int32_t clearing, int64_t* out_pairs, int64_t* n_pairs) {
    if (max_dim < 0 || max_dim > 3 || !counts || !order || !out_pairs || !n_pairs) {
        fph::set_error("fph_persistence_pairs: bad arguments");
        return FPH_EARG;
    }
    // global simplex id = offset[k] + row; rank = order[id]
    int64_t off[5] = {0, 0, 0, 0, 0};
    for (int k = 0; k <= max_dim; ++k) off[k + 1] = off[k] + counts[k];
    const int64_t n = off[max_dim + 1];
    if (n > 0x7fffffffLL) {
        fph::set_error("fph_persistence_pairs: more than 2^31 simplices");
        return FPH_EARG;
    }
    std::vector<int32_t> dim_of(n), id_of_rank(n);
    for (int k = 0; k <= max_dim; ++k)
        for (int64_t i = 0; i < counts[k]; ++i) {
            const int64_t r = order[off[k] + i];
            if (r < 0 || r >= n) {
                fph::set_error("fph_persistence_pairs: order is not a permutation");
                return FPH_EINTEGRITY;
            }
            dim_of[r] = k;
            id_of_rank[r] = (int32_t)(off[k] + i);
        }
    // boundary columns in rank space
    std::vector<std::vector<int32_t>> col(n);
    for (int64_t r = 0; r < n; ++r) {
        const int k = dim_of[r];
        if (k == 0) continue;
        const int64_t row = id_of_rank[r] - off[k];
        std::vector<int32_t>& c = col[r];
        c.reserve(k + 1);
        for (int j = 0; j <= k; ++j) {
            const int64_t f = facets[k][row * (k + 1) + j];
            c.push_back((int32_t)order[off[k - 1] + f]);
        }
        std::sort(c.begin(), c.end());
        if (c.back() >= r) {
            fph::set_error("face order violated at rank %lld", (long long)r);
            return FPH_EINTEGRITY;
        }
    }
    std::vector<int32_t> owner(n, -1);  // pivot row -> column
    std::vector<char> cleared(n, 0);
    std::vector<int32_t> tmp;
    auto reduce = [&](int64_t j) {
        if (cleared[j]) return;
        std::vector<int32_t>& c = col[j];
        while (!c.empty()) {
            const int32_t o = owner[c.back()];
            if (o < 0) break;
            sym_diff(c, col[o], tmp);
            c.swap(tmp);
        }
        if (!c.empty()) {
            owner[c.back()] = (int32_t)j;
            if (clearing) cleared[c.back()] = 1;
        }
    };
    if (clearing && max_dim > 0) {
        for (int k = max_dim; k >= 1; --k)
            for (int64_t r = 0; r < n; ++r)
                if (dim_of[r] == k) reduce(r);
    } else {
        for (int64_t r = 0; r < n; ++r) reduce(r);
    }
    int64_t np = 0;
    for (int64_t i = 0; i < n; ++i)
        if (owner[i] >= 0) {
            out_pairs[2 * np] = i;
            out_pairs[2 * np + 1] = owner[i];
            ++np;
        }
    *n_pairs = np;
    return FPH_OK;
}
