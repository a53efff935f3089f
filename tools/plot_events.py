#!/usr/bin/env python3
"""NEXT-2: queue-utilisation chart from a profiler export table (cf4ocl's ccl_plot_events,
P:59; Fig. 5).  Reads the tab-separated export of prng_prof_export
("queue<TAB>start_ns<TAB>end_ns<TAB>event name") and writes a plain SVG: one lane per queue,
one bar per event, colour per event name.

    python tools/plot_events.py events.tsv out.svg [--title "..."]
"""
import argparse
import html

COLORS = {"INIT_KERNEL": "#4c72b0", "RNG_KERNEL": "#55a868", "READ_BUFFER": "#c44e52", "OUT": "#8172b2"}
FALLBACK = ["#937860", "#da8bc3", "#8c8c8c", "#ccb974", "#64b5cd"]


def read_table(path):
    rows = []
    with open(path) as f:
        for line in f:
            q, a, b, n = line.rstrip("\n").split("\t")
            rows.append((q, int(a), int(b), n))
    return rows


def render(rows, title="", width=1200, lane_h=40):
    queues = []
    for q, _, _, _ in rows:
        if q not in queues:
            queues.append(q)
    order = {"Main": 0, "Comms": 1, "Host": 2}
    queues.sort(key=lambda q: order.get(q, 3))
    t0 = min(a for _, a, _, _ in rows) if rows else 0
    t1 = max(b for _, _, b, _ in rows) if rows else 1
    span = max(t1 - t0, 1)
    left, top = 90, 40
    plot_w = width - left - 20
    h = top + lane_h * len(queues) + 70
    names = []
    for _, _, _, n in rows:
        if n not in names:
            names.append(n)
    color = {n: COLORS.get(n, FALLBACK[i % len(FALLBACK)]) for i, n in enumerate(names)}
    out = [f'<svg xmlns="http://www.w3.org/2000/svg" width="{width}" height="{h}" font-family="sans-serif" '
           f'font-size="12">', f'<rect width="{width}" height="{h}" fill="white"/>',
           f'<text x="{left}" y="20" font-size="14">{html.escape(title)}</text>']
    for i, q in enumerate(queues):
        y = top + i * lane_h
        out.append(f'<text x="{left - 8}" y="{y + lane_h / 2 + 4}" text-anchor="end">{html.escape(q)}</text>')
        out.append(f'<rect x="{left}" y="{y + 4}" width="{plot_w}" height="{lane_h - 8}" fill="#f2f2f2"/>')
    for q, a, b, n in rows:
        y = top + queues.index(q) * lane_h
        x = left + (a - t0) / span * plot_w
        w = max((b - a) / span * plot_w, 0.5)
        out.append(f'<rect x="{x:.2f}" y="{y + 6}" width="{w:.2f}" height="{lane_h - 12}" fill="{color[n]}">'
                   f'<title>{html.escape(n)} {(b - a) / 1e6:.3f} ms</title></rect>')
    ya = top + lane_h * len(queues) + 18
    for k in range(6):
        x = left + k / 5 * plot_w
        out.append(f'<text x="{x:.1f}" y="{ya}" text-anchor="middle">{(span * k / 5) / 1e6:.1f} ms</text>')
    for i, n in enumerate(names):
        x = left + i * 160
        out.append(f'<rect x="{x}" y="{ya + 14}" width="12" height="12" fill="{color[n]}"/>')
        out.append(f'<text x="{x + 16}" y="{ya + 25}">{html.escape(n)}</text>')
    out.append("</svg>")
    return "\n".join(out) + "\n"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("table")
    ap.add_argument("svg")
    ap.add_argument("--title", default="")
    a = ap.parse_args()
    with open(a.svg, "w") as f:
        f.write(render(read_table(a.table), a.title))


if __name__ == "__main__":
    main()
