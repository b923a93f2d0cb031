// gd_pack.cpp -- the model packer.
//
// Takes trees in the reference's GbtNode form (models.hpp:35-43; any node
// order: level order from fit_gbt, preorder from load_model) and emits one
// 16-byte gd::PNode per reachable node, tree after tree, each tree laid out
// breadth-first from its root with the two children of every internal node
// in adjacent slots (so a node stores only its left-child index).  Leaves
// keep their original tree-local index for leaf-id output.
//
// The reference trusts its trees (predict_row indexes blindly,
// models.cpp:71-78); the packer rejects what would be undefined behaviour
// there: children out of range, a node reached twice (shared subtree or
// cycle), a split feature outside [0, n_cols).
#include <cstdio>
#include <string>
#include <vector>

#include "gd_host.hpp"

namespace gdh {

int pack_forest(const gd_forest_view& f, int32_t n_cols, std::vector<gd::PNode>& nodes,
                std::vector<int32_t>& roots, int32_t& max_depth) {
    nodes.clear();
    roots.clear();
    max_depth = 0;
    if (f.n_trees < 0) return set_error(GD_ERR_INVALID_ARGUMENT, "gbt model: negative tree count");
    if (f.n_trees > 0 && (!f.tree_offsets || !f.feature || !f.threshold || !f.left || !f.right || !f.leaf_value)) {
        return set_error(GD_ERR_INVALID_ARGUMENT, "gbt model: null node array");
    }
    std::vector<int32_t> pos, depth, queue;
    char buf[256];
    for (int32_t t = 0; t < f.n_trees; ++t) {
        const int64_t off = f.tree_offsets[t];
        const int64_t cnt = f.tree_offsets[t + 1] - off;
        if (cnt <= 0 || cnt > INT32_MAX) {
            std::snprintf(buf, sizeof(buf), "gbt tree %d: invalid node count", t);
            return set_error(GD_ERR_DATA, buf);
        }
        pos.assign(static_cast<size_t>(cnt), -1);
        depth.assign(static_cast<size_t>(cnt), 0);
        queue.clear();
        const int64_t base = static_cast<int64_t>(nodes.size());
        if (base + cnt > INT32_MAX) return set_error(GD_ERR_UNSUPPORTED, "gbt model: more than 2^31 nodes");
        roots.push_back(static_cast<int32_t>(base));
        nodes.push_back(gd::PNode{});
        pos[0] = static_cast<int32_t>(base);
        queue.push_back(0);
        for (size_t qi = 0; qi < queue.size(); ++qi) {
            const int32_t u = queue[qi];
            const int64_t k = off + u;
            gd::PNode pn{};
            if (f.feature[k] < 0) {
                pn.v = f.leaf_value[k];
                pn.feat = -1;
                pn.aux = u;
            } else {
                if (f.feature[k] >= n_cols) {
                    std::snprintf(buf, sizeof(buf), "gbt tree %d node %d: feature %d out of range (n_cols %d)", t, u,
                                  f.feature[k], n_cols);
                    return set_error(GD_ERR_DATA, buf);
                }
                const int32_t l = f.left[k], r = f.right[k];
                if (l < 0 || r < 0 || l >= cnt || r >= cnt || pos[l] >= 0 || pos[r] >= 0 || l == r) {
                    std::snprintf(buf, sizeof(buf), "gbt tree %d node %d: invalid children (%d, %d)", t, u, l, r);
                    return set_error(GD_ERR_DATA, buf);
                }
                const int32_t lp = static_cast<int32_t>(nodes.size());
                nodes.push_back(gd::PNode{});
                nodes.push_back(gd::PNode{});
                pos[l] = lp;
                pos[r] = lp + 1;
                depth[l] = depth[r] = depth[u] + 1;
                if (depth[l] > max_depth) max_depth = depth[l];
                pn.v = f.threshold[k];
                pn.feat = f.feature[k];
                pn.aux = lp;
                queue.push_back(l);
                queue.push_back(r);
            }
            nodes[static_cast<size_t>(pos[u])] = pn;
        }
    }
    return GD_OK;
}

}  // namespace gdh
