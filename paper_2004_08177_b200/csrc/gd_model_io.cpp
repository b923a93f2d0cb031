// gd_model_io.cpp -- "gpudvfs-model 1" reader feeding the packer directly.
//
// Restates load_model / load_model_file (models.cpp:639-714) over an
// in-memory token scan instead of std::istream extraction: leading '#'
// comment lines skipped (textio.hpp:39-44), then whitespace-separated tokens
// in the fixed order header / kind / target / encoding_ref / columns /
// (gbt: base, learning_rate, trees, tree N, node f thr l r leaf ...) or
// (linear: intercept, min_norm, coef name value ...).  Doubles are parsed
// with strtod (correctly rounded, so the %.17g written by save_model
// round-trips bit-exactly, models.cpp:611-633).  Error kinds and messages
// follow the reference: missing file -> missing_artifact_error
// "cannot open model '<path>'", malformed -> data_error "<path>: ...".
#include <cerrno>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "gd_host.hpp"

namespace gdh {
namespace {

struct Scanner {
    const char* p;
    const char* end;
    bool failed = false;

    bool next(std::string& tok) {
        if (failed) return false;
        while (p < end && (*p == ' ' || *p == '\n' || *p == '\t' || *p == '\r' || *p == '\f' || *p == '\v')) ++p;
        if (p >= end) {
            failed = true;
            return false;
        }
        const char* s = p;
        while (p < end && !(*p == ' ' || *p == '\n' || *p == '\t' || *p == '\r' || *p == '\f' || *p == '\v')) ++p;
        tok.assign(s, p);
        return true;
    }
    bool number(double& v) {
        std::string tok;
        if (!next(tok)) return false;
        char* e = nullptr;
        errno = 0;
        v = std::strtod(tok.c_str(), &e);
        if (e == tok.c_str() || *e != '\0') {
            failed = true;
            v = 0.0;
            return false;
        }
        return true;
    }
    template <typename I>
    bool integer(I& v) {
        std::string tok;
        if (!next(tok)) return false;
        char* e = nullptr;
        const long long x = std::strtoll(tok.c_str(), &e, 10);
        if (e == tok.c_str() || *e != '\0') {
            failed = true;
            v = 0;
            return false;
        }
        v = static_cast<I>(x);
        return true;
    }
};

}  // namespace

int parse_model_file(const char* path, gd_model& m) {
    const std::string origin(path ? path : "");
    FILE* fp = path ? std::fopen(path, "rb") : nullptr;
    if (!fp) return set_error(GD_ERR_MISSING_ARTIFACT, "cannot open model '" + origin + "'");
    std::string text;
    char buf[1 << 16];
    size_t got;
    while ((got = std::fread(buf, 1, sizeof(buf), fp)) > 0) text.append(buf, got);
    std::fclose(fp);

    // textio.hpp:39-44 skip_comment_lines
    size_t start = 0;
    while (start < text.size() && text[start] == '#') {
        const size_t nl = text.find('\n', start);
        start = nl == std::string::npos ? text.size() : nl + 1;
    }
    Scanner sc{text.data() + start, text.data() + text.size()};
    std::string tok, version;
    if (!sc.next(tok) || !sc.next(version) || tok != "gpudvfs-model" || version != "1") {
        return set_error(GD_ERR_DATA, origin + ": not a gpudvfs-model v1 file");
    }
    auto expect = [&](const char* want) -> bool { return sc.next(tok) && tok == want; };
    auto expect_err = [&](const char* want) {
        return set_error(GD_ERR_DATA, origin + ": expected '" + want + "' in model file");
    };

    std::string value;
    if (!expect("kind")) return expect_err("kind");
    sc.next(value);
    if (value == "gbt") m.kind = GD_KIND_GBT;
    else if (value == "ols") m.kind = GD_KIND_OLS;
    else if (value == "lasso") m.kind = GD_KIND_LASSO;
    else return set_error(GD_ERR_INVALID_ARGUMENT, "unknown model kind '" + value + "'");
    if (!expect("target")) return expect_err("target");
    sc.next(value);
    if (value == "energy") m.target = GD_TARGET_ENERGY;
    else if (value == "time") m.target = GD_TARGET_TIME;
    else return set_error(GD_ERR_INVALID_ARGUMENT, "unknown target '" + value + "' (expected energy or time)");
    if (!expect("encoding_ref")) return expect_err("encoding_ref");
    sc.next(value);
    size_t n = 0;
    if (!expect("columns")) return expect_err("columns");
    sc.integer(n);
    m.columns.clear();
    for (size_t i = 0; i < n; ++i) {
        if (!expect("column")) return expect_err("column");
        sc.next(value);
        m.columns.push_back(value);
    }
    m.n_cols = static_cast<int32_t>(m.columns.size());
    if (m.kind == GD_KIND_GBT) {
        if (!expect("base")) return expect_err("base");
        sc.number(m.base);
        if (!expect("learning_rate")) return expect_err("learning_rate");
        sc.number(m.lr);
        size_t trees = 0;
        if (!expect("trees")) return expect_err("trees");
        sc.integer(trees);
        m.offsets.assign(1, 0);
        m.feature.clear();
        m.threshold.clear();
        m.left.clear();
        m.right.clear();
        m.leaf.clear();
        for (size_t t = 0; t < trees; ++t) {
            if (!expect("tree")) return expect_err("tree");
            size_t count = 0;
            sc.integer(count);
            for (size_t k = 0; k < count; ++k) {
                if (!expect("node")) return expect_err("node");
                int32_t f = -1, l = -1, r = -1;
                double thr = 0.0, leaf = 0.0;
                sc.integer(f);
                sc.number(thr);
                sc.integer(l);
                sc.integer(r);
                sc.number(leaf);
                m.feature.push_back(f);
                m.threshold.push_back(thr);
                m.left.push_back(l);
                m.right.push_back(r);
                m.leaf.push_back(leaf);
            }
            m.offsets.push_back(static_cast<int64_t>(m.feature.size()));
        }
    } else {
        if (!expect("intercept")) return expect_err("intercept");
        sc.number(m.base);
        if (!expect("min_norm")) return expect_err("min_norm");
        int flag = 0;
        sc.integer(flag);
        m.coef.assign(m.columns.size(), 0.0);
        for (size_t j = 0; j < m.columns.size(); ++j) {
            if (!expect("coef")) return expect_err("coef");
            sc.next(value);
            sc.number(m.coef[j]);
            if (value != m.columns[j]) {
                return set_error(GD_ERR_DATA, origin + ": coefficient order mismatch at '" + value + "'");
            }
        }
    }
    if (sc.failed) return set_error(GD_ERR_DATA, origin + ": truncated model file");
    return GD_OK;
}

}  // namespace gdh
