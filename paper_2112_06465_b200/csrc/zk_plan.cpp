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
    // stages: subtrees of the same recursion with <= items / lanes leaves
    auto make_stages = [&](int32_t items) {
        std::vector<int32_t> stages;  // (b_lo, b_hi, l_lo, l_hi)
        const int32_t maxl = std::max<int32_t>(1, items / B.lanes);
        auto first_leaf = [&](int32_t pos) {  // first leaf starting at or after pos
            return (int32_t)(std::lower_bound(B.leaf_start.begin(), B.leaf_start.end(), pos) - B.leaf_start.begin());
        };
        std::vector<std::pair<int32_t, int32_t>> todo;  // explicit stack of (s, L), leftmost first
        if (L > 0 && !seq) todo.push_back({0, L});
        std::vector<std::pair<int32_t, int32_t>> ranges;
        while (!todo.empty()) {
            auto [s0, l0] = todo.back();
            todo.pop_back();
            const int32_t lo = first_leaf(s0), hi = first_leaf(s0 + l0);
            if (hi - lo <= maxl) {
                ranges.push_back({s0, l0});
                continue;
            }
            int32_t hh;
            if (B.lanes == 4) {
                hh = (l0 - l0 % 8) / 2;
            } else {
                hh = l0 / 2;
                hh -= hh % 8;
            }
            todo.push_back({s0 + hh, l0 - hh});  // right pushed first: left is processed first
            todo.push_back({s0, hh});
        }
        if (ranges.empty()) {  // L == 0 (head only) or a sequential leaf
            stages.insert(stages.end(), {0, 1 + std::max(L, 0), 0, nleaves});
        } else {
            for (size_t k = 0; k < ranges.size(); ++k) {
                const int32_t s0 = ranges[k].first, l0 = ranges[k].second;
                stages.insert(stages.end(), {k == 0 ? 0 : 1 + s0, 1 + s0 + l0, first_leaf(s0), first_leaf(s0 + l0)});
            }
        }
        return stages;
    };
    const std::vector<int32_t> stages = make_stages(kStageItems), stages16 = make_stages(kStageItems / 2);
    h.nstages[0] = (int32_t)(stages.size() / 4);
    h.nstages[1] = (int32_t)(stages16.size() / 4);
    size_t leaves_bytes = sizeof(int32_t) * 2 * (size_t)nleaves;
    size_t ops_bytes = sizeof(int32_t) * 4 * (size_t)cnt;
    size_t stages_bytes = sizeof(int32_t) * stages.size();
    size_t stages16_bytes = sizeof(int32_t) * stages16.size();
    h.leaves_off = (int32_t)((sizeof(PlanHeader) + 15) / 16 * 16);
    h.ops_off = (int32_t)((h.leaves_off + leaves_bytes + 15) / 16 * 16);
    h.stages_off[0] = (int32_t)((h.ops_off + ops_bytes + 15) / 16 * 16);
    h.stages_off[1] = (int32_t)((h.stages_off[0] + stages_bytes + 15) / 16 * 16);
    size_t total = (h.stages_off[1] + stages16_bytes + 15) / 16 * 16;
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
        std::memcpy(o + h.stages_off[0], stages.data(), stages_bytes);
        std::memcpy(o + h.stages_off[1], stages16.data(), stages16_bytes);
    }
    return total;
}

}  // namespace zk
