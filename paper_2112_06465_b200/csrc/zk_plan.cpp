// zk_plan.cpp -- host construction of pairwise-summation plans (see zk_plan.h).
#include "zk_plan.h"

#include <algorithm>
#include <cstring>
#include <vector>

namespace zk {

namespace {

struct Builder {
    int32_t leafmax, lanes;
    std::vector<int32_t> leaf_start, leaf_len;
    struct Inner { int32_t a, b, level; };
    std::vector<Inner> inner;   // internal node i has id nleaves_final + i (fixed up later)
    // node ids: leaves are tagged >= 0, internal nodes are tagged < 0 (-(i+1))
    std::vector<int32_t> level_of_leaf;

    int32_t rec(int32_t s, int32_t L, int32_t* level) {
        if (L <= leafmax) {
            leaf_start.push_back(s);
            leaf_len.push_back(L);
            *level = 0;
            return (int32_t)leaf_start.size() - 1;
        }
        int32_t h;
        if (lanes == 4) {
            h = (L - L % 8) / 2;       // CDOUBLE: n2 = n/2 - (n/2)%8 doubles, n = 2L
        } else {
            h = L / 2;                 // DOUBLE: n2 = n/2 - (n/2)%8
            h -= h % 8;
        }
        int32_t la, lb;
        int32_t a = rec(s, h, &la);
        int32_t b = rec(s + h, L - h, &lb);
        inner.push_back({a, b, std::max(la, lb) + 1});
        *level = std::max(la, lb) + 1;
        return -(int32_t)inner.size();
    }
};

}  // namespace

size_t build_plan(int32_t L, int32_t kind, void* out) {
    Builder B;
    B.lanes = (kind == kComplex) ? 4 : 8;
    B.leafmax = (kind == kComplex) ? 64 : 128;
    int32_t root = 0, rootlevel = 0;
    bool seq = L < B.lanes;
    if (L > 0) {
        if (seq) {
            B.leaf_start.push_back(0);
            B.leaf_len.push_back(L);
            root = 0;
        } else {
            root = B.rec(0, L, &rootlevel);
        }
    }
    int32_t nleaves = (int32_t)B.leaf_start.size();
    auto node_id = [&](int32_t tag) { return tag >= 0 ? tag : nleaves + (-tag - 1); };
    int32_t ninner = (int32_t)B.inner.size();
    // group internal nodes by level -> rounds
    int32_t maxlevel = 0;
    for (auto& in : B.inner) maxlevel = std::max(maxlevel, in.level);
    std::vector<int32_t> ops;  // (dst, a, b, 0)
    PlanHeader h;
    std::memset(&h, 0, sizeof(h));
    h.nrounds = maxlevel;
    int32_t cnt = 0;
    for (int32_t lv = 1; lv <= maxlevel; ++lv) {
        h.round_off[lv - 1] = cnt;
        for (int32_t i = 0; i < ninner; ++i) {
            if (B.inner[i].level != lv) continue;
            ops.push_back(nleaves + i);
            ops.push_back(node_id(B.inner[i].a));
            ops.push_back(node_id(B.inner[i].b));
            ops.push_back(0);
            ++cnt;
        }
    }
    h.round_off[maxlevel] = cnt;
    h.L = L;
    h.kind = kind;
    h.lanes = B.lanes;
    h.seq = seq ? 1 : 0;
    h.nleaves = nleaves;
    h.nnodes = nleaves + ninner;
    h.root = (L > 0) ? node_id(root) : 0;
    h.nops = cnt;
    for (int j = 0; j <= 129; ++j) {
        int k = 0;  // leaves are in ascending position order
        while (k < nleaves && 1 + B.leaf_start[k] + B.leaf_len[k] <= 32 * j) ++k;
        h.leaf_upto[j] = (int16_t)k;
    }
    size_t leaves_bytes = sizeof(int32_t) * 2 * (size_t)nleaves;
    size_t ops_bytes = sizeof(int32_t) * 4 * (size_t)cnt;
    h.leaves_off = (int32_t)((sizeof(PlanHeader) + 15) / 16 * 16);
    h.ops_off = (int32_t)((h.leaves_off + leaves_bytes + 15) / 16 * 16);
    size_t total = (h.ops_off + ops_bytes + 15) / 16 * 16;
    if (out) {
        char* o = static_cast<char*>(out);
        std::memset(o, 0, total);
        std::memcpy(o, &h, sizeof(h));
        int32_t* lv = reinterpret_cast<int32_t*>(o + h.leaves_off);
        for (int32_t i = 0; i < nleaves; ++i) {
            lv[2 * i] = B.leaf_start[i];
            lv[2 * i + 1] = B.leaf_len[i];
        }
        if (cnt) std::memcpy(o + h.ops_off, ops.data(), ops_bytes);
    }
    return total;
}

}  // namespace zk
