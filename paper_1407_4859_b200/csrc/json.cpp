// json.cpp -- see json.h.
#include "json.h"

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

namespace adha {
namespace json {

bool Value::has(const std::string& k) const { return find(k) != nullptr; }

const Value* Value::find(const std::string& k) const {
    if (kind != Object) return nullptr;
    for (auto& kv : obj)
        if (kv.first == k) return &kv.second;
    return nullptr;
}

const Value& Value::at(const std::string& k) const {
    const Value* v = find(k);
    if (!v) throw ParseError("missing key '" + k + "'");
    return *v;
}

double Value::as_num() const {
    if (kind != Number) throw ParseError("expected a number");
    return num;
}
const std::string& Value::as_str() const {
    if (kind != String) throw ParseError("expected a string");
    return str;
}
bool Value::as_bool() const {
    if (kind != Bool) throw ParseError("expected true/false");
    return b;
}
const std::vector<Value>& Value::as_arr() const {
    if (kind != Array) throw ParseError("expected an array");
    return arr;
}

namespace {
struct Parser {
    const char* p;
    const char* end;

    [[noreturn]] void error(const char* what) {
        throw ParseError(std::string("JSON: ") + what);
    }
    void ws() {
        while (p < end && (*p == ' ' || *p == '\t' || *p == '\n' || *p == '\r')) ++p;
    }
    bool lit(const char* s) {
        size_t n = std::strlen(s);
        if ((size_t)(end - p) >= n && std::memcmp(p, s, n) == 0) {
            p += n;
            return true;
        }
        return false;
    }
    static void put_utf8(std::string& out, uint32_t cp) {
        if (cp < 0x80) out += (char)cp;
        else if (cp < 0x800) { out += (char)(0xC0 | (cp >> 6)); out += (char)(0x80 | (cp & 0x3F)); }
        else if (cp < 0x10000) {
            out += (char)(0xE0 | (cp >> 12)); out += (char)(0x80 | ((cp >> 6) & 0x3F));
            out += (char)(0x80 | (cp & 0x3F));
        } else {
            out += (char)(0xF0 | (cp >> 18)); out += (char)(0x80 | ((cp >> 12) & 0x3F));
            out += (char)(0x80 | ((cp >> 6) & 0x3F)); out += (char)(0x80 | (cp & 0x3F));
        }
    }
    uint32_t hex4() {
        if (end - p < 4) error("bad \\u escape");
        uint32_t v = 0;
        for (int i = 0; i < 4; ++i) {
            char c = *p++;
            v <<= 4;
            if (c >= '0' && c <= '9') v |= (uint32_t)(c - '0');
            else if (c >= 'a' && c <= 'f') v |= (uint32_t)(c - 'a' + 10);
            else if (c >= 'A' && c <= 'F') v |= (uint32_t)(c - 'A' + 10);
            else error("bad hex digit");
        }
        return v;
    }
    std::string string() {
        if (p >= end || *p != '"') error("expected string");
        ++p;
        std::string out;
        while (p < end && *p != '"') {
            char c = *p++;
            if (c == '\\') {
                if (p >= end) error("bad escape");
                char e = *p++;
                switch (e) {
                    case '"': out += '"'; break;
                    case '\\': out += '\\'; break;
                    case '/': out += '/'; break;
                    case 'b': out += '\b'; break;
                    case 'f': out += '\f'; break;
                    case 'n': out += '\n'; break;
                    case 'r': out += '\r'; break;
                    case 't': out += '\t'; break;
                    case 'u': {
                        uint32_t cp = hex4();
                        if (cp >= 0xD800 && cp < 0xDC00 && end - p >= 6 && p[0] == '\\' && p[1] == 'u') {
                            p += 2;
                            uint32_t lo = hex4();
                            cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
                        }
                        put_utf8(out, cp);
                        break;
                    }
                    default: error("bad escape");
                }
            } else {
                out += c;
            }
        }
        if (p >= end) error("unterminated string");
        ++p;
        return out;
    }
    Value value(int depth) {
        if (depth > 200) error("nesting too deep");
        ws();
        if (p >= end) error("unexpected end");
        Value v;
        char c = *p;
        if (c == '{') {
            ++p;
            v.kind = Value::Object;
            ws();
            if (p < end && *p == '}') { ++p; return v; }
            for (;;) {
                ws();
                std::string k = string();
                ws();
                if (p >= end || *p != ':') error("expected ':'");
                ++p;
                v.obj.emplace_back(std::move(k), value(depth + 1));
                ws();
                if (p < end && *p == ',') { ++p; continue; }
                if (p < end && *p == '}') { ++p; break; }
                error("expected ',' or '}'");
            }
        } else if (c == '[') {
            ++p;
            v.kind = Value::Array;
            ws();
            if (p < end && *p == ']') { ++p; return v; }
            for (;;) {
                v.arr.push_back(value(depth + 1));
                ws();
                if (p < end && *p == ',') { ++p; continue; }
                if (p < end && *p == ']') { ++p; break; }
                error("expected ',' or ']'");
            }
        } else if (c == '"') {
            v.kind = Value::String;
            v.str = string();
        } else if (lit("true")) {
            v.kind = Value::Bool; v.b = true;
        } else if (lit("false")) {
            v.kind = Value::Bool; v.b = false;
        } else if (lit("null")) {
            v.kind = Value::Null;
        } else {
            char* q = nullptr;
            std::string tmp(p, std::min<size_t>(64, end - p));
            double d = std::strtod(tmp.c_str(), &q);
            if (q == tmp.c_str()) error("unexpected character");
            p += (q - tmp.c_str());
            v.kind = Value::Number;
            v.num = d;
        }
        return v;
    }
};
}  // namespace

Value parse(const std::string& text) {
    Parser ps{text.data(), text.data() + text.size()};
    Value v = ps.value(0);
    ps.ws();
    if (ps.p != ps.end) throw ParseError("JSON: trailing characters");
    return v;
}

std::string quote(const std::string& s) {
    std::string o = "\"";
    for (char c : s) {
        switch (c) {
            case '"': o += "\\\""; break;
            case '\\': o += "\\\\"; break;
            case '\n': o += "\\n"; break;
            case '\r': o += "\\r"; break;
            case '\t': o += "\\t"; break;
            default:
                if ((unsigned char)c < 0x20) {
                    char buf[8];
                    std::snprintf(buf, sizeof buf, "\\u%04x", (unsigned)(unsigned char)c);
                    o += buf;
                } else {
                    o += c;
                }
        }
    }
    return o + "\"";
}

std::string number(double v) {
    if (!std::isfinite(v)) return "null";
    char buf[40];
    for (int prec = 1; prec <= 17; ++prec) {
        std::snprintf(buf, sizeof buf, "%.*g", prec, v);
        if (std::strtod(buf, nullptr) == v) break;
    }
    return buf;
}

}  // namespace json
}  // namespace adha
